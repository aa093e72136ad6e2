# stream-K chain (B <= 8): parity + A/B bench
timeout 1500 python -m pytest tests/test_gpu_stack.py tests/test_gpu_attention.py tests/test_gpu_lm.py "tests/test_gpu_fullsize.py::test_stack_full_width_two_layers" tests/test_gpu_fullsize.py::test_stack_7b_width_chain_four_layers tests/test_gpu_comm.py::test_nccl_communicator_single_rank_in_graph -q -x --timeout 1200 > gpurun_out/sk_pytest.log 2>&1; echo "pytest exit $?"; grep -E "passed|failed|Error" gpurun_out/sk_pytest.log | tail -3
for v in 0 1; do for B in 2 8; do
  if [ $v = 1 ]; then export IFB_NO_MS_SK=1; else unset IFB_NO_MS_SK; fi
  timeout 120 python bench.py --batch $B --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nosk=$v B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"
done; done
unset IFB_NO_MS_SK
timeout 120 python bench.py --kv-pos 255 --batch 8 --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kv255 B=8', round(d['value'],1), 'tok/s')"
for m in 13b 70b; do timeout 300 python bench.py --model $m --batch 8 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m B=8', round(d['value'],1), 'tok/s')"; done
