# decode tokens/s sweep: batch sizes on 7B, then 13B / 70B at batch 1
for b in 1 2 4 8 16 32 64; do
  timeout 300 python bench.py --steps 20 --warmup 3 --batch $b --no-cpu-baseline 2>gpurun_out/sweep_b$b.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('7b B=$b', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms', round(d['hbm_gbs']), 'GB/s launches/step', d['gpu_launches']//d['steps'])" || tail -2 gpurun_out/sweep_b$b.err
done
for m in 13b 70b; do
  timeout 600 python bench.py --steps 10 --warmup 3 --model $m --no-cpu-baseline 2>gpurun_out/sweep_$m.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m B=1', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms', round(d['hbm_gbs']), 'GB/s frac', round(d['roofline']['frac'],3))" || tail -2 gpurun_out/sweep_$m.err
done
