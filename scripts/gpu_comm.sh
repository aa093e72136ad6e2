timeout 900 python -m pytest tests/test_gpu_comm.py -q -x --timeout 300 > gpurun_out/pytest_comm.log 2>&1; echo "exit $?"; tail -30 gpurun_out/pytest_comm.log
