# KV decode through the fused chain (B >= 2): parity (attention, LM/engine, stack) + KV bench + engine bench
timeout 1200 python -m pytest tests/test_gpu_attention.py tests/test_gpu_lm.py tests/test_gpu_stack.py -q -x --timeout 900 > gpurun_out/kvchain_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/kvchain_pytest.log
for P in 255 1023; do for B in 2 8 16; do
  timeout 300 python bench.py --kv-pos $P --batch $B --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pos=$P B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms', round(d['hbm_gbs']), 'GB/s launches/step', d['gpu_launches']//d['steps'])"
done; done
timeout 300 python scripts/engine_bench.py 2>&1 | tail -2
