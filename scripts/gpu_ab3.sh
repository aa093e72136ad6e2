# A/B decode-engine variant libraries: stack parity (SMALL + 7B), bench value, timeline
for v in "$@"; do
  lib=/root/repo/paper_2401_08294_b200/$v.so
  IFB_LIB_PATH=$lib timeout 600 python -m pytest tests/test_gpu_stack.py -q -x -k "decode and not batch64" 2>&1 | tail -1 | sed "s/^/$v tests: /"
  IFB_LIB_PATH=$lib timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>gpurun_out/ab_$v.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms frac', round(d['roofline']['frac'],3))"
  IFB_LIB_PATH=$lib timeout 120 python scripts/mk_timeline2.py 32 2>&1 | tail -8
done
