"""Phase/level attribution of the fused forward kernel from the -DDNLS_TRACE build.

usage: DNLS_LIB=trace python tools/trace.py [C2] ; prints cycles per phase (CTA 0).
Tags: 100 jac, 200 assemble, 300 factor..., 1000+l level start, 1100+l staged, 1200+l updates
done, 1300+l panels factored, 1999 factor end, 2000+l / 2100+l forward solve level (start /
staged), 3000+l / 3100+l backward solve, 400 retract start, 500 iteration end.
"""
import ctypes
import os
import sys
from collections import defaultdict

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


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = CONFIGS[name]
    B = int(os.environ.get("TRACE_B", cfg["B"]))
    N = int(os.environ.get("TRACE_N", cfg["N"]))
    topo = synth.cube_topology(N, dim=cfg["dim"], p=cfg["p"], mode=cfg["mode"], seed=0)
    data = synth.cube_batch(topo, B, seed=0)
    dev = torch.device("cuda", 0)
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in data.items()}
    solver = PoseGraphSolver(D.SE3 if cfg["dim"] == 3 else D.SE2, topo.num_poses, topo.edges, topo.prior_vars,
                             device=0, max_iterations=cfg["K"])
    buf = (ctypes.c_int64 * (2 * 8192))()
    n = ctypes.c_int32()
    for rep in range(2):
        _lib.lib().dnls_debug_trace(buf, 8192, ctypes.byref(n))   # reset
        solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], implicit=True)
        torch.cuda.synchronize()
        _lib.check(_lib.lib().dnls_debug_trace(buf, 8192, ctypes.byref(n)), "trace")
    arr = np.frombuffer(buf, dtype=np.int64)[:2 * n.value].reshape(-1, 2)
    tags, clk = arr[:, 0], arr[:, 1]
    dur = defaultdict(int)
    for i in range(len(tags) - 1):
        tg = int(tags[i])
        d = int(clk[i + 1] - clk[i])
        if tg in (100,):
            dur["jac"] += d
        elif tg == 200:
            dur["assemble"] += d
            dur["lin:zero"] += d
        elif tg == 210:
            dur["assemble"] += d
            dur["lin:jac"] += d
        elif tg == 220:
            dur["assemble"] += d
            dur["lin:scatter"] += d
        elif tg == 300:
            dur["factor:prologue"] += d
        elif tg == 900 or 5000 <= tg < 8000:
            dur["factor:forest"] += d
        elif tg == 950:
            dur["factor:forest->top"] += d
        elif tg == 3500:
            dur["bsolve:forest"] += d
        elif tg == 3999:
            dur["bsolve->retract"] += d
        elif 1000 <= tg < 1100:
            dur["factor:stage_in"] += d
        elif 1100 <= tg < 1150:
            dur[f"factor:U-own(l{tg - 1100})"] += d
            dur["factor:U-own(thread0)"] += d
        elif 1150 <= tg < 1160:
            dur["factor:U-waitsync"] += d
            dur[f"factor:U-waitsync(l{tg - 1150})"] += d
        elif 1160 <= tg < 1200:
            dur["factor:fwdrows"] += d
            dur[f"factor:fwdrows(l{tg - 1160})"] += d
        elif 1200 <= tg < 1300:
            dur[f"factor:F(l{tg - 1200})"] += d
            dur["factor:F"] += d
        elif 1300 <= tg < 1400:
            dur["factor:writeback"] += d
        elif tg == 1999:
            dur["factor->solve"] += d
        elif 2000 <= tg < 2100:
            dur["fsolve:stage_in"] += d
        elif 2100 <= tg < 2200:
            dur["fsolve:work"] += d
            dur[f"fsolve:work(l{tg - 2100})"] += d
        elif 3000 <= tg < 3100:
            dur["bsolve:stage_in"] += d
        elif 3100 <= tg < 3200:
            dur["bsolve:work"] += d
            dur[f"bsolve:work(l{tg - 3100})"] += d
        elif tg == 400:
            dur["retract"] += d
        elif tg == 500:
            dur["iter_end"] += d
    # forest tasks run by warp 0 (tags 5000+s start, 6000+s end) in the first factorisation
    starts = {}
    shown = 0
    for i in range(len(tags)):
        tg = int(tags[i])
        if 5000 <= tg < 6000:
            starts[tg - 5000] = clk[i]
        elif 6000 <= tg < 7000 and (tg - 6000) in starts and shown < 40:
            print(f"  forest task sn {tg - 6000}: {int(clk[i] - starts[tg - 6000])} cycles")
            shown += 1
    sub = defaultdict(int)
    names = {5000: "stage", 7001: "U", 7002: "fwdrows", 7003: "panel_factor", 7004: "trsv", 7005: "writeback"}
    for i in range(len(tags) - 1):
        tg = int(tags[i])
        key = 5000 if 5000 <= tg < 6000 else tg
        if key in names:
            sub[names[key]] += int(clk[i + 1] - clk[i])
    print("  warp-0 forest task breakdown (cycles, all factorisations):", dict(sub))
    total = int(clk[-1] - clk[0])
    print(f"{name}: total cycles (CTA 0) {total}  ({total / 1.9e3:.0f} us at 1.9 GHz), {len(tags)} trace points")
    for k, v in sorted(dur.items(), key=lambda kv: -kv[1]):
        print(f"  {k:28s} {v:12d}  {100.0 * v / total:5.1f}%")


if __name__ == "__main__":
    main()
