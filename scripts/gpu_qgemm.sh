timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "qgemm" --timeout 120 > gpurun_out/pytest_qgemm.log 2>&1; echo "exit $?"; tail -30 gpurun_out/pytest_qgemm.log
