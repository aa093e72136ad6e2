# precision margin of the chain at 7B width (4 layers, T = 8) with the hi + lo records
timeout 900 python -m pytest tests/test_gpu_fullsize.py::test_stack_7b_width_chain_four_layers -q -x -s --timeout 600 > gpurun_out/prec_pytest.log 2>&1; echo "pytest exit $?"; grep -E "normwise|passed|failed" gpurun_out/prec_pytest.log | tail -3
