ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 1 -c 1 -o gpurun_out/prof_unit python scripts/mk_timeline.py gemv 131072 4096 > gpurun_out/ncu_unit.log 2>&1
tail -1 gpurun_out/ncu_unit.log
