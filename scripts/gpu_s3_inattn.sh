# in-engine KV attention (B = 1): parity (attention + LM/engine tests) then bench A/B
timeout 600 python -m pytest tests/test_gpu_attention.py -q -x --timeout 300 > gpurun_out/inattn_pytest.log 2>&1; echo "pytest attention exit $?"; grep -E "passed|failed|Error|assert" gpurun_out/inattn_pytest.log | head -8
timeout 600 python -m pytest tests/test_gpu_lm.py -q -x --timeout 300 > gpurun_out/inattn_pytest2.log 2>&1; echo "pytest lm exit $?"; tail -1 gpurun_out/inattn_pytest2.log
for v in 0 1; do for P in 255 1023; do
  if [ $v = 1 ]; then export IFB_NO_MK_ATTN=1; else unset IFB_NO_MK_ATTN; fi
  timeout 120 python bench.py --kv-pos $P --batch 1 --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no_in_attn=$v pos=$P B=1', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms launches/step', d['gpu_launches']//d['steps'])"
done; done
