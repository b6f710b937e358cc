./tools/fp64lat
for r in "" "2,2,0,2,0,64,0" "2,3,0.5,4,0.3,64,0.2" "3,4,0.6,8,0.4,64,0.3"; do
  for c in C2 C4; do
    echo "RELAX=$r $c"; DNLS_RELAX=$r timeout 120 python tools/stage_times.py $c 10 2>&1 | tail -1
  done
done
