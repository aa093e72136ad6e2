for t in 1 6; do for B in 2 3 4 5 6; do
  IFB_MK_TMAX=$t timeout 300 python bench.py --batch $B --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tmax=$t B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"
done; done
