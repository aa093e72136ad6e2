# B=1 KV decode launch list (pos 255): engine partial launches vs attention kernels
timeout 300 python bench.py --kv-pos 255 --batch 1 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-160
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_mk|rope|attn" --launch-skip 200 -c 97 --csv --log-file gpurun_out/kv1_launches.csv python bench.py --kv-pos 255 --batch 1 --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu $?"
