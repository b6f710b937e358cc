set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python tools/shard_check.py /tmp/shard > gpurun_out/r2b_shard.txt 2>&1; tail -5 gpurun_out/r2b_shard.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/r2b_c5.json 2> gpurun_out/r2b_c5.err
cat gpurun_out/r2b_c5.json; tail -3 gpurun_out/r2b_c5.err
