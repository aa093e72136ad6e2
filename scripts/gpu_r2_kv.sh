# NEXT-1 KV decode: parity (attention, LM/engine, stack-kv) then the bench at pos 255 / 1023, B = 1 / 2 / 8
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_lm.py -q -x 2>&1 | tail -3
for P in 255 1023; do for B in 1 2 8; do
  timeout 300 python bench.py --kv-pos $P --batch $B --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pos=$P B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms', round(d['hbm_gbs']), 'GB/s launches/step', d['gpu_launches']//d['steps'])"
done; done
timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-150
timeout 300 python scripts/engine_bench.py 2>&1 | tail -1
