# chain: per-token RMS partial sums spread over a warp; parity + bench
timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_attention.py -q -x --timeout 600 > gpurun_out/rms_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/rms_pytest.log
for B in 2 8 16; do timeout 120 python bench.py --batch $B --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"; done
