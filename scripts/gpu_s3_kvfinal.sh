# final KV decode + serving engine numbers (7B, pos 255 / 1023, B = 1 / 2 / 8 / 16)
python -c "import torch; torch.zeros(1).cuda()"
for P in 255 1023; do for B in 1 2 8 16; do
  timeout 300 python bench.py --kv-pos $P --batch $B --steps 30 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pos=$P B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms launches/step', d['gpu_launches']//d['steps'])"
done; done
timeout 300 python scripts/engine_bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('engine', d['tokens_per_s'], 'tok/s; verify K=4', d['verify_K4_ms'], 'ms')"
