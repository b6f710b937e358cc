# timing ablation (development builds): forward time with one phase skipped (results invalid)
for v in abl skipu skipfwd skipf skipbs skipjac; do for c in C2 C4; do echo -n "$v $c "; DNLS_LIB=$v timeout 200 python tools/stage_times.py $c 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['forward_us'],1))"; done; done
