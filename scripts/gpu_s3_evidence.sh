# round-2 session-3 evidence: GPU suite, smoke, bench, batch sweep, launch list, ncu captures, reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 1500 > gpurun_out/s3_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/s3_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/s3_smoke.log
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/s3_bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/s3_bench.log | cut -c1-200
bash scripts/gpu_sweep.sh > gpurun_out/s3_sweep.txt 2>&1; cat gpurun_out/s3_sweep.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 3 -c 1 -o gpurun_out/s3_decode_mk python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu mk $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ms_chain -c 40 --csv --log-file gpurun_out/s3_chain_launches.csv python bench.py --batch 8 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu chain list $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ms_chain -s 3 -c 1 -o gpurun_out/s3_chain_gu python bench.py --batch 8 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu chain full $?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/s3_reference.log 2>&1; tail -1 gpurun_out/s3_reference.log | cut -c1-200
