IFB_LIB_PATH=/root/repo/paper_2401_08294_b200/libif_poll.so timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_fullsize.py -q -k "not prefill and not quantize" 2>&1 | tail -2
for v in libif_b200 libif_poll; do
  lib=/root/repo/paper_2401_08294_b200/$v.so
  for m in 7b 13b 70b; do
    IFB_LIB_PATH=$lib timeout 600 python bench.py --model $m --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $m', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],3), 'launches', d['gpu_launches'])"
  done
  IFB_MODEL=7b IFB_LIB_PATH=$lib timeout 300 python scripts/mk_timeline2.py 32 2>&1 | grep -A6 "^kind"
done
bash scripts/gpu_r2_sanitize.sh
