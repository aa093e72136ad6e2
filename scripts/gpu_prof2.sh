python scripts/prof_sweep.py 4096
python scripts/prof_sweep.py 11008
ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 3 -c 1 -o gpurun_out/prof_mk_o python scripts/prof_gemv.py --reps 1 --copies 4 --shapes o > gpurun_out/ncu_o.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 3 -c 1 -o gpurun_out/prof_mk_gu python scripts/prof_gemv.py --reps 1 --copies 4 --shapes gu > gpurun_out/ncu_gu.log 2>&1
tail -2 gpurun_out/ncu_o.log
