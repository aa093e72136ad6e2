# usage: bash scripts/gpu_r2_ab2.sh "models" lib1 lib2 ...   (bench only)
models=$1; shift
for v in "$@"; do
  lib=/root/repo/paper_2401_08294_b200/$v.so
  for m in $models; do
    IFB_LIB_PATH=$lib timeout 600 python bench.py --model $m --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $m', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms frac', round(d['roofline']['frac'],3))"
  done
done
