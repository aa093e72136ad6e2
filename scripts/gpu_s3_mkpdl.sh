# engine partial launches with PDL (KV decode B=1): parity + bench A/B
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_lm.py tests/test_gpu_stack.py -q -x --timeout 600 > gpurun_out/mkpdl_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/mkpdl_pytest.log
for v in 0 1; do for P in 255 1023; do
  if [ $v = 1 ]; then export IFB_MK_NOPDL=1; else unset IFB_MK_NOPDL; fi
  timeout 300 python bench.py --kv-pos $P --batch 1 --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nopdl=$v pos=$P B=1', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms')"
done; done
