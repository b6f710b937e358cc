"""Per-element equality of a 2-rank bench run and the 1-rank run (SURVEY.md §8(e) pin P12): runs
bench.py --config C5 --batch 64 at --gpus 1 and --gpus 2 (gloo, both ranks on cuda:0 when the box has
one GPU) with --dump-shard, then compares theta_K / objectives per global element (bitwise) and the
all-reduced gradients (1e-12)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = sys.argv[1] if len(sys.argv) > 1 else "/tmp/shard"
common = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C5", "--batch", "64", "--steps", "3",
          "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--no-factor-roofline"]
one_gpu = "--share-gpu" if len(sys.argv) < 3 or sys.argv[2] != "multi" else None
r1 = subprocess.run(common + ["--gpus", "1", "--dump-shard", out + "1"], capture_output=True, text=True)
print(r1.stdout[-400:], r1.stderr[-2000:])
extra = ["--dist-backend", "gloo", "--share-gpu"] if one_gpu else []
r2 = subprocess.run(common + ["--gpus", "2", "--dump-shard", out + "2"] + extra, capture_output=True, text=True)
print(r2.stdout[-600:], r2.stderr[-2000:])
a = np.load(out + "1.rank0.npz")
s = [np.load(out + f"2.rank{r}.npz") for r in range(2)]
P2 = np.concatenate([x["poses"] for x in s])
O2 = np.concatenate([x["obj"] for x in s])
assert [(int(x["b0"]), int(x["b1"])) for x in s] == [(0, 32), (32, 64)]
print("theta_K bitwise equal:", np.array_equal(a["poses"], P2), " objectives bitwise equal:", np.array_equal(a["obj"], O2))
g1, g2 = a["grads"], s[0]["grads"]
print("reduced grads rel diff:", float(np.max(np.abs(g1 - g2)) / np.max(np.abs(g1))),
      " ranks agree:", np.array_equal(s[0]["grads"], s[1]["grads"]))
assert np.array_equal(a["poses"], P2) and np.array_equal(a["obj"], O2)
assert np.max(np.abs(g1 - g2)) <= 1e-12 * np.max(np.abs(g1))
print("SHARD CHECK OK")
