"""Host-side logic of multi-step training: which actors hold a tied parameter
and which one updates it (taskgraph.py:349-361: the lowest stage's actor)."""
from paper_2412_14374_b200 import comms as C
from paper_2412_14374_b200 import ir as I
from paper_2412_14374_b200 import schedules as S
from paper_2412_14374_b200 import taskgraph as T
from paper_2412_14374_b200.executor import tied_holders


def _tg(p, s):
    return T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)


def test_gpt_tied_embedding_holders():
    cfg = I.GPTConfig(layers=4, d_model=64, n_heads=2, d_ff=128, vocab=96, seq_len=16,
                      microbatch_size=2, yields=(2, 3, 5), yield_every=6)
    tg = _tg(I.derive_backward(I.partition_stages(I.build_gpt(cfg))), S.one_f_one_b(4, 4))
    assert tied_holders(tg) == [("w0", 0, {0: "wbuf:w0:a0", 3: "wbuf:w0:a3"})]
    C.plan_pipeline(tg)


def test_untied_and_single_actor_have_no_holders():
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=4, width=4, microbatch_size=2, yield_every=1))))
    assert tied_holders(_tg(p, S.one_f_one_b(4, 4))) == []
    pt = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=4, width=4, microbatch_size=2, yield_every=4, tied_weights=True))))
    assert tied_holders(_tg(pt, S.gpipe(1, 2))) == []


def test_interleaved_tied_weight_on_one_actor_twice():
    # stages 0 and 3 of an interleaved P=2 V=2 layout live on actors 0 and 1
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=4, width=4, microbatch_size=2, yield_every=1, tied_weights=True))))
    (q, low, hs), = tied_holders(_tg(p, S.interleaved_1f1b(2, 4, 2)))
    assert low == 0 and sorted(hs) == [0, 1]
