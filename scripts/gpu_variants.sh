for v in libif_b200 libif_v11_8 libif_v7_8 libif_v11_4; do
  echo "== $v"
  IFB_LIB_PATH=/root/repo/paper_2401_08294_b200/$v.so python scripts/prof_sweep.py 4096 2>&1 | tail -2
  IFB_LIB_PATH=/root/repo/paper_2401_08294_b200/$v.so timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms', round(d['hbm_gbs']), 'GB/s')"
done
IFB_LIB_PATH=/root/repo/paper_2401_08294_b200/libif_b200.so python scripts/mk_timeline.py stack 2
