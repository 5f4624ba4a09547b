#!/bin/bash
# One GPU round trip for a kernel change: the GPU parity suite, per-phase device times of a C5
# and a C2 search (tools/acg_sweep.py, env variants as arguments), and with LAUNCHES=1 an ncu
# launch list (kernel durations) of one C2 and one C5 search.  Output: gpurun_out/quick.txt
out=gpurun_out/quick.txt
: > $out
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> $out
fi
for c in ${CONFIGS:-C5 C2}; do timeout 300 python tools/acg_sweep.py $c "${@:-NONE=0}" >> $out 2>&1; done
if [ -n "$LAUNCHES" ]; then
  for c in C2 C5; do
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      python tools/one_search.py $c seeded 1 > gpurun_out/launch_$c.csv 2>/dev/null
    python tools/launch_summary.py gpurun_out/launch_$c.csv >> $out 2>&1 || true
  done
fi
cat $out
