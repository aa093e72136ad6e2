# NEXT-2/3/4 GPU checks + cost-model calibration + bench launch list
set -x
timeout 900 python -m pytest tests/test_gpu_lm.py -q -rf -s 2>&1 | tail -15
timeout 2400 python scripts/calibrate_cost.py --steps 30 > gpurun_out/calib.log 2>&1; echo "calib exit $?"; tail -5 gpurun_out/calib.log
cp profiles/r2_cost_calibration.json gpurun_out/ 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
