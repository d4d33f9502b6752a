make -s >/dev/null 2>&1
GQSA_FIX_LOCAL=0 timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 200 python tools/sanitize_small.py > gpurun_out/racecheck2.log 2>&1; echo racecheck rc=$?; tail -2 gpurun_out/racecheck2.log
grep -E "^=========     (Read|Write) Thread" gpurun_out/racecheck2.log | sed 's/Thread ([0-9,]*)//; s/+0x[0-9a-f]*//' | sort | uniq -c | head -20
