# U/F cost vs shared-memory residency (trace build): C2 at several smem budgets, and N=128
for kb in 223 150 90; do echo "SMEM_KB=$kb"; DNLS_SMEM_KB=$kb DNLS_LIB=trace timeout 200 python tools/trace.py C2 2>&1 | sed -n 2,8p; done
for kb in 223 60; do echo "N=128 SMEM_KB=$kb"; TRACE_N=128 DNLS_SMEM_KB=$kb DNLS_LIB=trace timeout 200 python tools/trace.py C2 2>&1 | sed -n 2,8p; done
