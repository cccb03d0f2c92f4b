"""Debug: multi-rank (loopback) fused ring on slabs vs one rank, full residual histories."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
from paper_1308_5626_b200 import inputs, pspgmres as P
from test_gpu_multirank import multi_steps, single_steps, FUSED_MODES

case, mode, nr = sys.argv[1], sys.argv[2], int(sys.argv[3])
if case == "C2s":
    prob = inputs.c2(n=64, d=1, steps=2)
else:
    prob = inputs.Problem("C4s", inputs.OperatorSpec(3, "cell_diff", (20, 18, 16), 2e-4,
                                                     field=np.exp(np.random.default_rng(5).standard_normal(20 * 18 * 16))),
                          np.random.default_rng(6).uniform(-1, 1, 20 * 18 * 16), 30, 1e-8, 3, 2, 32, 1000)
m = multi_steps(torch, P, prob, nr, 1, FUSED_MODES[mode])
s = single_steps(torch, P, prob, 1, FUSED_MODES[mode])
hm, hs = m["reps"][0]["resid_history"], s["reps"][0]["resid_history"]
print("iters", m["reps"][0]["iterations"], s["reps"][0]["iterations"])
for i in range(min(len(hm), len(hs), 45)):
    print(i, hm[i], hs[i], abs(hm[i] - hs[i]) / max(hs[i], 1e-300))
print("u diff", np.linalg.norm(m["u"] - s["u"]) / np.linalg.norm(s["u"]))
