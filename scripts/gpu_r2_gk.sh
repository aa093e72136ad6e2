timeout 1200 python -m pytest tests/test_gpu_engine_schemes.py tests/test_gpu_kernels.py tests/test_gpu_stack.py -q -x 2>&1 | tail -4
for sc in Q3H_B64 Q4_B32 Q4_B64 Q8_B64 Q8_B32 Q2_B32 Q2_B64 Q3_B32 Q3_B64 Q5_B64 Q6_B64; do
  timeout 600 python bench.py --scheme $sc --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sc', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms frac', round(d['roofline']['frac'],3), 'launches', d['gpu_launches'])"
done
