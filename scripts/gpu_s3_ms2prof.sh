# ncu --set full of the gate/up qgemv_ms2 launch (B = 8) + bench B=8 stdout
timeout 300 python bench.py --batch 8 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_b8.log 2>&1; tail -1 gpurun_out/bench_b8.log | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qgemv_ms2 -s 2 -c 1 -o gpurun_out/s3_ms2_gu python bench.py --batch 8 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_ms2.log 2>&1; echo "ncu exit $?"
