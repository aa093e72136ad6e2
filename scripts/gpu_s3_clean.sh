# after removing the knock-out knobs from the chain kernel: parity + bench
timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_attention.py tests/test_gpu_lm.py -q -x --timeout 600 > gpurun_out/clean_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/clean_pytest.log
for B in 2 8 16; do timeout 120 python bench.py --batch $B --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms', d['roofline']['kernel'][:30])"; done
