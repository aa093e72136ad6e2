# prefill qGEMM with the f32x2 Q3H dequant: parity (qgemm kernels + full-size prefill shapes) + timing
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -x --timeout 900 -k "qgemm or prefill" > gpurun_out/pf_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pf_pytest.log
timeout 900 python scripts/prof_prefill.py --schemes Q3H:64 --M 512 2>&1 | tail -8
timeout 900 python scripts/prof_prefill.py --schemes Q3H:64 --M 2048 2>&1 | tail -4
