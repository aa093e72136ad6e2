timeout 1200 python -m pytest tests/test_gpu_stack.py tests/test_gpu_attention.py tests/test_gpu_fullsize.py tests/test_gpu_lm.py -q -x 2>&1 | tail -4
for B in 8 16 32 64; do
  timeout 600 python bench.py --batch $B --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('7b B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms', 'launches', d['gpu_launches'])"
done
