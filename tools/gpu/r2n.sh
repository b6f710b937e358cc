# persistent factorisation with dynamic scheduling; hybrid split level sweep
python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
DNLS_BL_SPLIT=12 python -m pytest tests/test_gpu_bl.py -x -q 2>&1 | tail -2
run() { tag=$1; shift; env "$@" python bench.py --config $C --interleave 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-factor-roofline > gpurun_out/r2n_$tag.json 2> gpurun_out/r2n_$tag.err
  python -c "import json; d=json.load(open('gpurun_out/r2n_$tag.json')); r=d['roofline']; print('$tag', round(d['value']), round(d['ms_per_step'],2), round(r['kernel_ms'],3), round(r['frac'],4), r.get('forward_frac'))" || tail -3 gpurun_out/r2n_$tag.err; }
C=C5
run c5_p0 DNLS_BL_PERSIST=0
for sp in 0 6 12 20 26 34; do run c5_s$sp DNLS_BL_SPLIT=$sp; done
run c5_s12_ct8 DNLS_BL_SPLIT=12 DNLS_BL_COLTASK=8
run c5_s12_gw32 DNLS_BL_SPLIT=12 DNLS_BL_PERSIST=32
run c5_s12_gw8 DNLS_BL_SPLIT=12 DNLS_BL_PERSIST=8
run c5_s12_ch16 DNLS_BL_SPLIT=12 DNLS_BL_CH=16,2
run c5_s12_ch64 DNLS_BL_SPLIT=12 DNLS_BL_CH=64,1
C=C4
run c4_p0 DNLS_BL_PERSIST=0
run c4_p0u0 DNLS_BL_PERSIST=0 DNLS_BL_UPD=0
for sp in 0 12 26; do run c4_s$sp DNLS_BL_SPLIT=$sp; done
run c4_s12_gw8 DNLS_BL_SPLIT=12 DNLS_BL_PERSIST=8
run c4_s12_gw16 DNLS_BL_SPLIT=12 DNLS_BL_PERSIST=16
