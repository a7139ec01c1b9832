"""Experiment: does running the cfg2 evaluation as two concurrent halves (two host threads, two
streams, 25 shots x 3 Hz each, separate helm_ops) hide the fixed per-cycle latency? Prints the
wall time of one call over all 150 pairs vs two concurrent half calls (after warm-up), and
checks that the two halves add up to the whole."""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1703_09268_b200 import api  # noqa: E402

p = synth.cfg2()
grid, pml = api.Grid.of(p), api.Pml(v_ref=3000.0)
opts = api.SolveOpts(rtol=1e-6)
d, _ = api.fwi_forward(grid, p.m_true, p.freqs, p.src, p.rec, pml, api.C128, api.SolveOpts(rtol=1e-8), max_rhs=150)
ns = len(p.src)


def whole():
    fg, _ = api.fwi_misfit_grad(grid, p.m, p.freqs, p.src, p.rec, d, pml, api.C128, opts, max_rhs=150)
    return fg


def halves(k=2):
    outs = [None] * k
    cuts = [ns * i // k for i in range(k + 1)]

    def work(i):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            fg, _ = api.fwi_misfit_grad(grid, p.m, p.freqs, p.src, p.rec, d, pml, api.C128, opts,
                                        max_rhs=(cuts[i + 1] - cuts[i]) * len(p.freqs), src_range=(cuts[i], cuts[i + 1]),
                                        stream=st)
        st.synchronize()
        outs[i] = fg
    th = [threading.Thread(target=work, args=(i,)) for i in range(k)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return sum(outs[1:], outs[0])


for name, fn in (("whole", whole), ("halves2", lambda: halves(2)), ("halves3", lambda: halves(3)),
                 ("whole", whole), ("halves2", lambda: halves(2)), ("halves3", lambda: halves(3))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(name, round((time.perf_counter() - t0) * 1e3, 1), "ms", float(r[0]), flush=True)
a, b = whole().cpu().numpy(), halves(2).cpu().numpy()
print("rel diff whole vs halves", np.linalg.norm(a - b) / np.linalg.norm(a))
