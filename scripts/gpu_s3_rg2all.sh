# 256-row tiles wherever the cost model prefers them (qkv + gate/up at 7B): parity + A/B
timeout 1200 python -m pytest tests/test_gpu_stack.py tests/test_gpu_attention.py "tests/test_gpu_fullsize.py::test_stack_full_width_two_layers" tests/test_gpu_fullsize.py::test_stack_7b_width_chain_four_layers -q -x --timeout 900 > gpurun_out/rg2all_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/rg2all_pytest.log
python -c "import torch; torch.zeros(1).cuda()"
for v in 0 1 0; do for B in 2 8; do
  if [ $v = 1 ]; then export IFB_NO_MS_RG2=1; else unset IFB_NO_MS_RG2; fi
  timeout 200 python bench.py --batch $B --steps 50 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('norg2=$v B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"
done; done
python scripts/ms_timeline.py 8 2 2>&1 | tail -4
