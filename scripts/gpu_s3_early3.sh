# early start only for the 3.5-bit engine: k-bit engine parity + Q8_B64 / Q3H bench
timeout 900 python -m pytest tests/test_gpu_engine_schemes.py tests/test_gpu_stack.py -q -x --timeout 600 > gpurun_out/early3_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/early3_pytest.log
for sc in Q8_B64 Q3H_B64; do timeout 300 python bench.py --scheme $sc --steps 50 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sc', round(d['value'],1), 'tok/s frac', round(d['roofline']['frac'],4))"; done
