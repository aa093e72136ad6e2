# Round evidence: GPU tests, bench line, launch list, ncu --set full of the three hot kernels,
# batch sweep, prefill schemes.  Every step under its own timeout.
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu_r1.log 2>&1; tail -1 gpurun_out/pytest_gpu_r1.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
cat gpurun_out/bench_r1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 2 -c 1 -o gpurun_out/decode_mk_r1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemm_tc -s 2 -c 1 -o gpurun_out/qgemm_tc_r1 python scripts/prof_prefill.py --schemes Q3H:64 --gemm-only > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemv_tc -s 72 -c 1 -o gpurun_out/qgemv_tc_r1 python scripts/prof_tc_sweep.py 8 > /dev/null 2>&1
timeout 900 bash scripts/gpu_sweep.sh > gpurun_out/sweep_r1.txt 2>&1
for M in 64 512; do timeout 300 python scripts/prof_prefill.py --M $M 2>&1 | tail -20; done > gpurun_out/prefill_r1.txt
timeout 120 python scripts/mk_timeline2.py 32 > gpurun_out/timeline_r1.txt 2>&1
ls gpurun_out/
