"""Per-level cycle attribution of the first factorisation of the per-element forward kernel (-DDNLS_TRACE
build, CTA 0 / cluster rank 0): for every supernodal level the update gathers (tags 1100 -> 1160), the
forward rows + group barrier (1160 -> 1200) and the dense panels + barrier (1200 -> 1300).

usage: DNLS_LIB=trace python tools/trace_levels.py C3r [K]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("DNLS_LIB", "trace")

import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2207_09442_b200 import _lib  # noqa: E402
from paper_2207_09442_b200 import dnls as D  # noqa: E402
from paper_2207_09442_b200.layer import PoseGraphSolver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = CONFIGS[name]
topo = synth.cube_topology(cfg["N"], dim=cfg["dim"], p=cfg["p"], mode=cfg["mode"], seed=0)
data = synth.cube_batch(topo, cfg["B"], seed=0)
dev = torch.device("cuda", 0)
t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in data.items() if k != "gt"}
opt = {"lm": D.LM, "gn": D.GN}[cfg["opt"]]
# one CTA per element: the trace buffer lives in the main translation unit (the clustered kernel has its own)
solver = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=K,
                         optimizer=opt, cluster_ctas=1)
buf = (ctypes.c_int64 * (2 * 8192))()
n = ctypes.c_int32()
_lib.lib().dnls_debug_trace(buf, 8192, ctypes.byref(n))
solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], implicit=True)
torch.cuda.synchronize()
_lib.check(_lib.lib().dnls_debug_trace(buf, 8192, ctypes.byref(n)), "trace")
arr = np.frombuffer(buf, dtype=np.int64)[:2 * n.value].reshape(-1, 2)
tags, clk = arr[:, 0].tolist(), arr[:, 1].tolist()
st = solver.stats
print(f"{name}: {n.value} trace points, levels {st['num_levels']}, supernodes {st['num_supernodes']}")
pos = {}
first_end = tags.index(1999) if 1999 in tags else len(tags)
for i in range(first_end):
    pos.setdefault(tags[i], i)
tot = {"U": 0, "fwd": 0, "F": 0}
rows = []
for lv in range(st["num_levels"]):
    a, b, c, d = (pos.get(1100 + lv), pos.get(1160 + lv), pos.get(1200 + lv), pos.get(1300 + lv))
    if None in (a, b, c, d):
        continue
    u, f, p = clk[b] - clk[a], clk[c] - clk[b], clk[d] - clk[c]
    tot["U"] += u
    tot["fwd"] += f
    tot["F"] += p
    rows.append((lv, u, f, p))
T = sum(tot.values())
print(f"first factorisation: {T} cycles ({T / 1.965e3:.0f} us): " +
      ", ".join(f"{k} {100 * v / max(T, 1):.1f}%" for k, v in tot.items()))
for lv, u, f, p in rows:
    print(f"  level {lv:3d}: U {u:9d}  fwd+sync {f:9d}  F+sync {p:9d}")
