# round-2 evidence refresh -> gpurun_out/ev_* (copied to profiles/ by hand)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/ev_bench.log 2>&1; tail -1 gpurun_out/ev_bench.log
bash scripts/gpu_sweep.sh > gpurun_out/ev_sweep.txt 2>&1
for sc in Q4_B32 Q4_B64 Q8_B64 Q8_B32 Q2_B32 Q2_B64 Q3_B32 Q3_B64 Q5_B64 Q6_B64; do
  timeout 600 python bench.py --scheme $sc --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sc', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms frac', round(d['roofline']['frac'],3), 'launches/step', d['gpu_launches']//d['steps'])"
done > gpurun_out/ev_schemes.txt 2>&1
for m in tensor tensor4 hybrid layer; do timeout 300 python scripts/tp_engine_check.py $m 3 2>&1 | tail -1; done > gpurun_out/ev_tp.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 500 -c 200 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qgemv_ms --launch-skip 2 -c 1 -o gpurun_out/ev_qgemv_ms python bench.py --batch 8 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu ms $?"
timeout 900 ncu --set full --clock-control none -k regex:decode_mk -c 1 -o gpurun_out/ev_decode_mk_q4 python bench.py --scheme Q4_B32 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu q4 $?"
timeout 900 ncu --set full --clock-control none -k regex:decode_mk -c 1 -o gpurun_out/ev_decode_mk_70b python bench.py --model 70b --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu 70b $?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_reference.log 2>&1; tail -1 gpurun_out/ev_reference.log | cut -c1-300
