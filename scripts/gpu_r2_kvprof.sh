# launch list of one KV decode step (7B, pos 255, B=1): per-kernel device durations
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_mk|attn|rope_append" -c 300 --csv --log-file gpurun_out/kv_launches.csv \
  python bench.py --kv-pos 255 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/kv_prof_bench.log 2>&1
tail -2 gpurun_out/kv_prof_bench.log | cut -c1-200
