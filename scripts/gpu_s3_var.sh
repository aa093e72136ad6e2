# chain occupancy variants (B = 8, 16): V=0 (2 CTAs/SM, ring 8) vs V=1 (3 CTAs/SM, ring 4)
for v in 0 1; do for B in 8 16; do
IFB_MS_VAR=$v timeout 300 python bench.py --batch $B --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/var${v}_$B.log 2>&1; tail -1 gpurun_out/var${v}_$B.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('V=$v B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"
done
IFB_MS_VAR=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ms_chain" -c 40 --csv --log-file gpurun_out/var${v}_launches.csv python bench.py --batch 8 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
