# chain: h loads of the o/down epilogue hoisted before the stores; parity + B sweep + timeline
timeout 900 python -m pytest tests/test_gpu_stack.py -q -x --timeout 600 > gpurun_out/emit_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/emit_pytest.log
for B in 2 8 16; do timeout 120 python bench.py --batch $B --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_b$B.log 2>&1; tail -1 gpurun_out/bench_b$B.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"; done
python scripts/ms_timeline.py 8 3 2>&1 | tail -5
