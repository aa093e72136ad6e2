# Prefill evidence after the wide-tile change: full GPU tests, bench line, ncu of the
# prefill qGEMM (wide tile), per-scheme prefill at M = 64 / 512 / 2048.
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu_r1b.log 2>&1; tail -1 gpurun_out/pytest_gpu_r1b.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err
cat gpurun_out/bench_r1b.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemm_tc -s 2 -c 1 -o gpurun_out/qgemm_tc_r1b python scripts/prof_prefill.py --schemes Q3H:64 --gemm-only > /dev/null 2>&1
for M in 64 512; do timeout 300 python scripts/prof_prefill.py --M $M 2>&1 | tail -20; done > gpurun_out/prefill_r1b.txt
timeout 300 python scripts/prof_prefill.py --M 2048 --schemes Q3H:64,Q4:32,Q8:64 > gpurun_out/prefill_r1b_2048.txt 2>&1
ls gpurun_out/ | grep r1b
