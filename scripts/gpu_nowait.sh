for v in libif_b200 libif_NOWAIT libif_NOWAIT8 libif_R8; do
IFB_LIB_PATH=/root/repo/paper_2401_08294_b200/$v.so python scripts/prof_sweep.py 4096 > gpurun_out/sw_$v.txt 2>&1; echo "$v $(tail -1 gpurun_out/sw_$v.txt)"
done
