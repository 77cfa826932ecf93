"""Host-side pieces of full per-stage rematerialisation (CPU): the stash-bytes
accounting (RunStats.peak_stash_bytes) and the policy names, which follow the
reference's simulator (simulator.py:48, :64-65, :144-149)."""
import pytest

torch = pytest.importorskip("torch")

from paper_2412_14374_b200 import executor as E  # noqa: E402
from paper_2412_14374_b200.device import Act  # noqa: E402


def test_policy_names_match_the_reference_simulator():
    assert (E.REMAT_NONE, E.REMAT_FULL) == ("none", "full-per-stage")


def test_stash_bytes_counts_each_tensor_once():
    a = torch.zeros(4, 8)                      # 128 B
    act = Act(torch.zeros(2, 8, dtype=torch.bfloat16))  # 32 B
    act.saved["ln"] = (a, torch.zeros(3))      # a again (not recounted) + 12 B
    stash = {"x": act, "h": a, "idx": torch.zeros(5, dtype=torch.int32), "meta": 3}
    assert E._stash_bytes(stash) == 128 + 32 + 12 + 20


def test_remat_stash_counts_the_kept_feeds_not_the_parameters():
    feeds = {"x": torch.zeros(16, dtype=torch.bfloat16)}
    params = {"w": torch.zeros(1024)}
    assert E._stash_bytes({"__remat__": (feeds, params)}) == 32


def test_retained_feeds_are_kept_by_reference_without_saved():
    """Feeds are kept by reference (nothing rewrites a feed before its backward in
    the same step); an Act is re-wrapped so the forward's saved tensors are not
    retained (the replay recomputes them)."""
    t = torch.arange(6.0)
    act = Act(torch.ones(3))
    act.saved["k"] = torch.zeros(100)
    rt, ra = E._retained(t), E._retained(act)
    assert rt is t and ra is not act and ra.t is act.t and ra.saved == {}
    assert E._retained(5) == 5
