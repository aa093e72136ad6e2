# decode engine check: stack/gemv GPU tests, per-phase timeline, short bench
timeout 600 python -m pytest tests/test_gpu_stack.py tests/test_gpu_kernels.py -q -x --timeout 300 > gpurun_out/pytest_mk.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_mk.log; grep -E "^E |Error|assert" gpurun_out/pytest_mk.log | head -10
timeout 120 python scripts/mk_timeline2.py 32 2>&1 | tail -7
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms', round(d['hbm_gbs']), 'GB/s', 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1))"
