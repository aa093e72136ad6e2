# decode_mk: start staging a phase input once all but E CTAs signalled (parity tags catch late words)
for E in 0 4 16 48 0; do
  IFB_MK_EARLY=$E timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('early=$E', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms frac', round(d['roofline']['frac'],4))"
done
IFB_MK_EARLY=16 timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_tp_engine.py tests/test_gpu_engine_schemes.py -q -x --timeout 600 > gpurun_out/early_pytest.log 2>&1; echo "pytest(early=16) exit $?"; tail -1 gpurun_out/early_pytest.log
