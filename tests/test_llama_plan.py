"""Llama-style (C5) graph through the planner on CPU: stage layout, the
non-adjacent skip channels for the position / token inputs, deadlock-free
plan, deterministic JSON, and the model-FLOP convention."""
import pytest

from paper_2412_14374_b200 import comms as C
from paper_2412_14374_b200 import ir as I
from paper_2412_14374_b200 import schedules as S
from paper_2412_14374_b200 import taskgraph as T


def plan(P, M, layers=14, V=1):
    cfg = I.LlamaConfig(layers=layers, d_model=256, n_heads=4, n_kv_heads=2, d_ff=512,
                        vocab=1000, seq_len=64, microbatch_size=1, yield_every=2)
    p = I.derive_backward(I.partition_stages(I.build_llama(cfg)))
    s = S.one_f_one_b(P, M) if V == 1 else S.interleaved_1f1b(P, M, V)
    tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
    return cfg, tg, C.plan_pipeline(tg)


def test_c5_layout_8_stage_skip_channels():
    cfg, tg, cp = plan(8, 16)
    assert cfg.num_stages == 8
    # positions feed every block, token ids the head: stage 0 sends to all stages
    for s in range(1, 8):
        assert (0, s) in cp.channels
    C.check_deadlock_free(cp)
    assert cp.to_json_str() == plan(8, 16)[2].to_json_str()


def test_llama_flops_convention():
    cfg = I.LlamaConfig(layers=32, d_model=4096, n_heads=32, n_kv_heads=8, d_ff=14336,
                        vocab=128256, seq_len=4096, microbatch_size=1)
    # C5 51.47 GFLOP/token
    assert cfg.flops_per_token() / 1e9 == pytest.approx(51.47, rel=2e-3)


def test_llama_config_validation():
    with pytest.raises(I.GraphError):
        I.LlamaConfig(layers=2, d_model=96, n_heads=4, n_kv_heads=3, d_ff=8, vocab=8,
                      seq_len=8, microbatch_size=1)
