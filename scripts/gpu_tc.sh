timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_stack.py -q -x --timeout 300 > gpurun_out/pytest_tc.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_tc.log; grep -E "^E |Error" gpurun_out/pytest_tc.log | head -8
for M in 64 512; do timeout 300 python scripts/prof_prefill.py --M $M --schemes Q3H:64,Q4:32 2>&1 | tail -4; done
bash scripts/gpu_sweep.sh
