# per-phase split sweep of the final chain (B = 8): IFB_MS_SPLITS="qkv,o,gu,down" (0 = cost model)
python -c "import torch; torch.zeros(1).cuda()"
for sp in "0,0,0,0" "0,4,0,0" "0,6,0,0" "0,12,0,0" "0,16,0,0" "0,0,0,6" "0,0,0,12" "0,0,0,16" "2,0,0,0" "4,0,0,0" "0,0,0,0"; do
  IFB_MS_SPLITS=$sp timeout 200 python bench.py --batch 8 --steps 50 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splits=$sp', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"
done
