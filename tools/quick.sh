#!/bin/bash
# One GPU round trip for a kernel change: the GPU parity suite, then per-phase device times
# of a C5 and a C2 search (tools/acg_sweep.py, default knobs unless given as arguments).
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/quick_tests.txt
for c in C5 C2; do timeout 300 python tools/acg_sweep.py $c "${@:-NONE=0}"; done
cat gpurun_out/quick_tests.txt
