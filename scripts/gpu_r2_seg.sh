timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_fullsize.py tests/test_gpu_kernels.py -q 2>&1 | tail -3
for v in libif_b200 libif_head; do
  lib=/root/repo/paper_2401_08294_b200/$v.so
  for m in 7b 13b 70b; do
    IFB_LIB_PATH=$lib timeout 600 python bench.py --model $m --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $m', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms frac', round(d['roofline']['frac'],3))"
  done
done
