ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 2 -c 1 -o gpurun_out/prof_mk_stack python scripts/mk_timeline.py stack 4 > gpurun_out/ncu_mk_stack.log 2>&1
tail -2 gpurun_out/ncu_mk_stack.log
