"""Host-side layout of the peer-memory channels (executor._slot_layout): one
flag word per message first, then one 256-byte-aligned slot per message in
the plan's order, sized from the message's wire layout."""
import torch

import bench
from paper_2412_14374_b200.executor import _slot_layout, _wire_meta_fn
from paper_2412_14374_b200.device import MODES


def test_c2_four_stage_slots():
    cfg, tg, cp = bench.build_plan(4, bench.C2, 8)
    meta = _wire_meta_fn(tg, MODES["bf16"])
    for key, bids in cp.channels.items():
        slots, total = _slot_layout(bids, meta)
        assert len(slots) == len(bids)
        assert slots[0][0] >= 4 * len(bids) and slots[0][0] % 256 == 0
        prev_end = 0
        for (off, shape, dtype, nb), bid in zip(slots, bids):
            assert off % 256 == 0 and off >= prev_end
            assert nb == torch.empty(shape, dtype=dtype, device="meta").numel() * \
                torch.empty((), dtype=dtype).element_size()
            prev_end = off + nb
        assert total >= prev_end
    # activations 0 -> 1: eight bf16 [8192, 768] boundary tensors
    slots, _ = _slot_layout(cp.channels[(0, 1)], meta)
    assert [s[1] for s in slots] == [(8192, 768)] * 8 and slots[0][2] == torch.bfloat16
    # the token skip 0 -> 3 is int32, the commuted tied-embedding gradient 3 -> 0 fp32
    assert _slot_layout(cp.channels[(0, 3)], meta)[0][0][2] == torch.int32
    assert _slot_layout(cp.channels[(3, 0)], meta)[0][0][2] == torch.float32
