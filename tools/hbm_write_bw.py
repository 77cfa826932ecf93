"""HBM write-only bandwidth (pc_fill and torch zero_ over 50-400 MB): the
ceiling for output-heavy epilogues.  usage: python tools/hbm_write_bw.py"""
import torch, sys
sys.path.insert(0, '/root/repo')
from paper_2412_14374_b200 import _lib
st = torch.cuda.current_stream().cuda_stream
for mb in (50, 100, 400):
    n = mb * 2**20 // 4
    t = torch.empty(n, device="cuda")
    for _ in range(3):
        _lib.call("pc_fill", _lib.PC_F32, n, 0.0, t.data_ptr(), st)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        _lib.call("pc_fill", _lib.PC_F32, n, 0.0, t.data_ptr(), st)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"pc_fill {mb} MB: {ms*1e3:.1f} us, {mb*2**20/ms/1e6:.0f} GB/s")
    s.record()
    for _ in range(20):
        t.zero_()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"torch zero_ {mb} MB: {ms*1e3:.1f} us, {mb*2**20/ms/1e6:.0f} GB/s")
