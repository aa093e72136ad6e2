# chain ring depth 12 (NT = 1): parity + bench
timeout 600 python -m pytest tests/test_gpu_stack.py -q -x --timeout 300 -k "chain or small" > gpurun_out/depth_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/depth_pytest.log
for B in 2 8; do timeout 200 python bench.py --batch $B --steps 50 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"; done
