for B in 1 8; do timeout 300 python tools/trace_tc.py --batch $B 2>&1 | tail -6; done
