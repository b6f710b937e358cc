# two CTAs per SM (256 threads, 128 registers, <= 110 KB shared memory each) vs the default
for c in C4 C2; do
  echo -n "default $c "; timeout 200 python tools/stage_times.py $c 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['forward_us'],1), round(d['backward_us'],1))"
  for kb in 110 100 80; do echo -n "nt256x2 smem=$kb $c "; DNLS_LIB=nt256x2 DNLS_SMEM_KB=$kb timeout 200 python tools/stage_times.py $c 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['forward_us'],1), round(d['backward_us'],1))"; done
done
