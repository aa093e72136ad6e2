# stream-K chain: per-kernel launch list (B = 8) + bench A/B
timeout 300 python -m pytest tests/test_gpu_stack.py -q -x --timeout 300 -k chain > gpurun_out/sk2_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/sk2_pytest.log
for v in 0 1; do for B in 8; do
  if [ $v = 1 ]; then export IFB_NO_MS_SK=1; else unset IFB_NO_MS_SK; fi
  timeout 120 python bench.py --batch $B --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nosk=$v B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"
done; done
unset IFB_NO_MS_SK
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"ms_chain" -c 9 --csv --log-file gpurun_out/sk_launches.csv python bench.py --batch 8 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu $?"
