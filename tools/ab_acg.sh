#!/bin/bash
# A/B of the R_co kernels on C2 (run on the GPU box): parity subset, then bench lines.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_distributed.py -x -q \
    -k "autocorr or golden or edge or egs or strips_gpu" 2>&1 | tail -2 > gpurun_out/ab_tests.txt
for v in "" "TMATCH_ACG_THREADS=128" "TMATCH_ACF=column"; do
  f=gpurun_out/acg_$(echo "$v" | tr "=" "_").json
  env $v timeout 300 python bench.py --no-cpu-baseline --steps 200 > $f 2>/dev/null
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2] or 'default', round(d['ms_per_step'],4), round(d['phases_ms_per_step']['autocorr_u8'],4), d['result']['best_rho'], d['result']['h_e'])" $f "$v"
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_acg -c 2 \
      -o gpurun_out/$NCU python tools/prep_only.py C2 > gpurun_out/acg_ncu.log 2>&1
  tail -1 gpurun_out/acg_ncu.log
fi
cat gpurun_out/ab_tests.txt
