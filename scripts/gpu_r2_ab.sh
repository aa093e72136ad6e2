# usage: bash scripts/gpu_r2_ab.sh lib1 lib2 ...  (parity of the engine + 7B/70B bench + 7B timeline)
for v in "$@"; do
  lib=/root/repo/paper_2401_08294_b200/$v.so
  IFB_LIB_PATH=$lib timeout 900 python -m pytest tests/test_gpu_stack.py -q -x -k "decode and not batch64" 2>&1 | tail -1 | sed "s/^/$v tests: /"
  for m in 7b 70b; do
    IFB_LIB_PATH=$lib timeout 600 python bench.py --model $m --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $m', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms frac', round(d['roofline']['frac'],3))"
  done
  IFB_MODEL=7b IFB_LIB_PATH=$lib timeout 300 python scripts/mk_timeline2.py 32 2>&1 | grep -A5 "^kind"
done
