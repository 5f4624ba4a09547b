set -x
python bench.py > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err
for c in C1 C2 C3 C4 C6; do l=$(echo $c | tr 'C' 'c'); python bench.py --config $c > gpurun_out/r02_bench_$l.json 2> gpurun_out/r02_bench_$l.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_c5_reference_arm.json 2> gpurun_out/ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c5.csv python tools/one_search.py C5 seeded 2 > gpurun_out/one_search.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -c 40 -o gpurun_out/r02_c5_full python tools/one_search.py C5 seeded 1 > gpurun_out/ncu_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c4_batch.csv python tools/one_batch.py C4 > gpurun_out/one_batch_c4.log 2>&1
ls -la gpurun_out | tail -20
