python scripts/prof_gemv.py --reps 20 --copies 8 2>&1 | tee gpurun_out/prof_events.txt
ncu --set full --clock-control none --import-source on -k regex:qgemv_q3h64 -s 2 -c 1 -o gpurun_out/prof_qkv python scripts/prof_gemv.py --reps 1 --copies 2 --shapes qkv > gpurun_out/ncu_qkv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:qgemv_q3h64 -s 2 -c 1 -o gpurun_out/prof_down python scripts/prof_gemv.py --reps 1 --copies 2 --shapes down > gpurun_out/ncu_down.log 2>&1
tail -3 gpurun_out/ncu_qkv.log
