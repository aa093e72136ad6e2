bash scripts/gpu_ab3.sh libif_if1 libif_if2 libif_if5 2>&1 | grep -E "tok/s|^sum|tests"
ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 2 -c 1 -o gpurun_out/prof_mk_v1 python scripts/mk_timeline.py stack 4 > gpurun_out/ncu_mk.log 2>&1
tail -2 gpurun_out/ncu_mk.log
