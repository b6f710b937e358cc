timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in nt256 "" nt512; do for c in C2 C4; do echo "variant=$v $c"; DNLS_LIB=$v timeout 200 python tools/stage_times.py $c 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v,1) for k,v in d.items() if k.endswith('_us')})"; done; done
