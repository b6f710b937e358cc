"""Measured fp64 peaks for the roofline denominators: cuBLAS DGEMM 8192^3 through
torch.matmul (library number, best of 5 and back to back for ~3 s) plus the hand DFMA / DMMA probes of
tools/fp64_peak.cu.  Writes one JSON line (committed as profiles/r2_fp64_peak.json)."""
import json
import os
import subprocess
import sys
import time

import torch

HERE = os.path.dirname(os.path.abspath(__file__))


def dgemm(n=8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    t0 = time.time()
    cnt = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 3.0:
        torch.matmul(a, b)
        cnt += 1
        if cnt % 4 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / cnt
    fl = 2.0 * n ** 3
    return fl / best / 1e9, fl / sus / 1e9


if __name__ == "__main__":
    burst, sustained = dgemm()
    exe = os.path.join(HERE, "fp64_peak")
    if not os.path.exists(exe):
        subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", exe,
                        os.path.join(HERE, "fp64_peak.cu")], check=True)
    probe = json.loads(subprocess.run([exe], capture_output=True, text=True, check=True).stdout)
    out = {"dgemm_tflops": burst, "dgemm_tflops_sustained": sustained, **probe,
           "gpu": torch.cuda.get_device_name(0),
           "how": "torch.matmul fp64 8192^3 (cuBLAS DGEMM), best of 5 and back to back ~3 s; hand DFMA "
                  "(8 independent chains/thread) and DMMA m8n8k4 (4 accumulators/warp) over 148x8 CTAs x 256 threads"}
    print(json.dumps(out))
    sys.stdout.flush()
