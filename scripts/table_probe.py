"""Config-4 batched Goodput table timing (device-resident traces, CUDA events)."""
import os, sys, tempfile, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2407_13126_b200 import planner, scenario as SC, workloads as W
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
work = tempfile.mkdtemp()
p = SC.Problem(SC.load_scenario(W.write_scenario(W.c2_spec(400000, steps=600, windows=1), work, "c4")), 0)
rng = np.random.default_rng(0)
traces = np.stack([W.mmpp_trace([40.0, 120.0, 12.0, 10.0], p.S, 400000 + k) for k in range(64)]).astype(np.int32)
traces = traces[rng.integers(0, 64, size=B)]  # B traces (resampled from 64 generated)
d_arr = torch.from_numpy(traces).cuda()
d_ub = torch.empty((B, p.S + 1), dtype=torch.float64, device="cuda")
d_best = torch.empty((B, p.S), dtype=torch.float64, device="cuda")
with planner.Planner(0) as pl:
    n_opt = len(pl.enumerate(p)["config"])
    st = torch.cuda.Stream()
    pl.lib.mgs_set_stream(pl.h, st.cuda_stream)
    torch.cuda.set_stream(st)
    for _ in range(2):
        npar = pl.goodput_table_batch_device(p, d_arr.data_ptr(), B, d_best.data_ptr(), d_ub.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    K = 5
    for _ in range(K):
        pl.goodput_table_batch_device(p, d_arr.data_ptr(), B, d_best.data_ptr(), d_ub.data_ptr())
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    ub_h, _ = pl.goodput_table_batch(p, traces[:4])
print("B %d M %d S %d |O| %d pareto %d: %.3f ms/batch, %.3g ref cells/s, %.3g scanned cells/s, ub0 %.6f" % (
    B, p.M, p.S, n_opt, npar, ms, B * p.S * n_opt / ms * 1e3, B * p.S * npar / ms * 1e3, ub_h[0, 0]))
