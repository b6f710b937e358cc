DNLS_LIB=trace timeout 600 python tools/trace_levels.py C3r 1 2>&1 | tail -45
DNLS_LIB=trace timeout 600 python tools/trace_levels.py C3 1 2>&1 | tail -45
