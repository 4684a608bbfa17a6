"""Two-stream concurrency probe for the bench workload (configs[3], both species): one block-diagonal
handle on one stream (the bench), two single-species handles one after the other on one stream, and
the two handles on two streams (their GEMMs and combination passes free to overlap).  Timing only."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

wl = W.config(3)
pb = wl.problems
vs = [torch.from_numpy(np.ascontiguousarray(W.as_flat(p.vs[0]))).cuda() for p in pb]
ells, tau = pb[0].ells, pb[0].tau
blk = PhiKS([p.A for p in pb])
sep = [PhiKS(p.A) for p in pb]
outs_b = [torch.empty_like(vs[0]) for _ in range(6)]
outs_s = [[torch.empty_like(vs[0]) for _ in range(3)] for _ in range(2)]
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(step, reps=10):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def block_step():
    blk.apply(tau, ells, vs, outs=outs_b)


def seq_step():
    for k in range(2):
        sep[k].apply(tau, ells, [vs[k]], outs=outs_s[k])


def two_stream_step():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    for k, s in enumerate((s0, s1)):
        s.wait_event(ev)
        sep[k].apply(tau, ells, [vs[k]], outs=outs_s[k], stream=s)
    for s in (s0, s1):
        e = torch.cuda.Event()
        e.record(s)
        cur.wait_event(e)


res = {"block_one_stream_ms": timeit(block_step), "two_handles_one_stream_ms": timeit(seq_step),
       "two_handles_two_streams_ms": timeit(two_stream_step)}
print(json.dumps(res))
