# RoPE/append fused into the attention kernel at T = 1: parity + KV bench A/B
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_lm.py tests/test_gpu_stack.py -q -x --timeout 600 > gpurun_out/rf2_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/rf2_pytest.log
python -c "import torch; torch.zeros(1).cuda()"
for v in 0 1; do for P in 255 1023; do
  if [ $v = 1 ]; then export IFB_NO_ROPE_FUSE=1; else unset IFB_NO_ROPE_FUSE; fi
  timeout 200 python bench.py --kv-pos $P --batch 1 --steps 50 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nofuse=$v pos=$P B=1', round(d['value'],1), 'tok/s launches/step', d['gpu_launches']//d['steps'])"
done; done
unset IFB_NO_ROPE_FUSE
timeout 300 python scripts/engine_bench.py 2>&1 | tail -1 | cut -c1-160
