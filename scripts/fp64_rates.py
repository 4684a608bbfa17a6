"""DMMA (kind 0) and DFMA (kind 1) fp64 throughput on one B200 (fp64_peak_kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, time
from paper_2210_07667_b200 import fp64_peak_launch
sink = torch.empty(148*8*256, dtype=torch.float64, device="cuda")
for kind in (0, 1):
    fp64_peak_launch(kind, 148*4, 200, sink)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fl = fp64_peak_launch(kind, 148*8, 20000, sink); e1.record(); torch.cuda.synchronize()
    print(kind, "TFLOP/s %.2f" % (fl / (e0.elapsed_time(e1) * 1e-3) / 1e12))
