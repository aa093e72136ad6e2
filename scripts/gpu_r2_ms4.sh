for v in libif_b200 libif_ms3 libif_ms4; do
 for B in 8 16 32; do
  IFB_LIB_PATH=/root/repo/paper_2401_08294_b200/$v.so timeout 600 python bench.py --batch $B --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"
 done
done
