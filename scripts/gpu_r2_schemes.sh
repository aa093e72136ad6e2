# batch-1 7B decode for every scheme (engine for Q3H_B64, per-layer generic path otherwise) + cost calibration
for sc in Q3H_B64 Q4_B32 Q4_B64 Q8_B64 Q8_B32 Q2_B32 Q3_B32 Q5_B64 Q6_B64 Q2_B64; do
  timeout 600 python bench.py --scheme $sc --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sc', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms frac', round(d['roofline']['frac'],3), 'launches', d['gpu_launches'])"
done
timeout 2400 python scripts/calibrate_cost.py --steps 30 > gpurun_out/calib.log 2>&1; echo "calib exit $?"; cp profiles/r2_cost_calibration.json gpurun_out/
