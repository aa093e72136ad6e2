# decode_mk early-start threshold on 13B / 70B and two k-bit schemes (B = 1)
python -c "import torch; torch.zeros(1).cuda()"
for m in 13b 70b; do for E in 0 16 32; do
  IFB_MK_EARLY=$E timeout 300 python bench.py --model $m --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m early=$E', round(d['value'],1), 'tok/s frac', round(d['roofline']['frac'],4))"
done; done
for sc in Q4_B32 Q8_B64; do for E in 0 16; do
  IFB_MK_EARLY=$E timeout 300 python bench.py --scheme $sc --steps 50 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sc early=$E', round(d['value'],1), 'tok/s frac', round(d['roofline']['frac'],4))"
done; done
