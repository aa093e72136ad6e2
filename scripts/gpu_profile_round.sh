set -x
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
cat gpurun_out/bench_r1.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 2 -c 1 -o gpurun_out/decode_mk_r1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:qgemm_tc -s 2 -c 1 -o gpurun_out/qgemm_tc_r1 python scripts/prof_prefill.py --schemes Q3H:64 --gemm-only > /dev/null 2>&1
ls -la gpurun_out/
