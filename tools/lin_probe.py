"""Cycles of the linearisation segments (CTA 0, thread 0) in k_forward, probe build:
DNLS_LIB=probe python tools/lin_probe.py [C2]"""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("DNLS_LIB", "probe")
import synth
from bench import CONFIGS
from paper_2207_09442_b200 import _lib, dnls as D
from paper_2207_09442_b200.layer import PoseGraphSolver
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
topo = synth.cube_topology(cfg["N"], dim=cfg["dim"], p=cfg["p"], mode=cfg["mode"], seed=0)
data = synth.cube_batch(topo, cfg["B"], seed=0)
t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in data.items()}
s = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=cfg["K"])
L = _lib.lib()
f = L.dnls_debug_probe
f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)()
for rep in range(3):
    f(buf, 1)
    s.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], implicit=True)
    torch.cuda.synchronize()
f(buf, 0)
n = cfg["K"] + 1
names = ["zero+sync", "slots", "slot-barrier wait", "pose gather+max", "finish: barrier", "finish: sums"]
for i, nm in enumerate(names):
    print(f"{nm:22s} {buf[i] / n:10.0f} cycles per linearisation")
