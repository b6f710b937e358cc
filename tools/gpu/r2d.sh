set -x
python -m pytest tests/test_gpu_train.py tests/test_gpu_parity.py -x -q 2>&1 | tail -5
( time python -m pytest tests/test_gpu_fullsize.py -x -q --durations=10 ) 2>&1 | tail -20
mkdir -p gpurun_out/sanitizer
for c in c1 c2 cluster lm unroll dlm; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $c > gpurun_out/sanitizer/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(tail -2 gpurun_out/sanitizer/${tool}_${c}.log | tr '\n' ' ')"
  done
done
python -m paper_2207_09442_b200.train --poses 1024 --batch 256 --epochs 20 > gpurun_out/r2d_train_c4.json 2>&1; tail -2 gpurun_out/r2d_train_c4.json
