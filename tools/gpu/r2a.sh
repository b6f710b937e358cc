set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2a_c5.json 2> gpurun_out/r2a_c5.err
python tools/stage_times.py C4 10 > gpurun_out/r2a_stage_c4.json 2>&1
python tools/stage_times.py C5 5 > gpurun_out/r2a_stage_c5.json 2>&1
python - <<'PY' > gpurun_out/r2a_fp64peak.txt 2>&1
import torch,time
a=torch.randn(8192,8192,dtype=torch.float64,device='cuda');b=torch.randn_like(a)
for _ in range(3): c=a@b
torch.cuda.synchronize()
best=1e9
for _ in range(5):
    s=torch.cuda.Event(enable_timing=True);e=torch.cuda.Event(enable_timing=True)
    s.record();c=a@b;e.record();torch.cuda.synchronize();best=min(best,s.elapsed_time(e))
print("dgemm 8192^3 ms",best,"TFLOP/s",2*8192**3/best/1e9)
PY
cat gpurun_out/r2a_c5.json gpurun_out/r2a_stage_c4.json gpurun_out/r2a_stage_c5.json gpurun_out/r2a_fp64peak.txt
