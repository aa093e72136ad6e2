# ncu --set full of the four chain kernels of one layer (B = 8): launches 2..5 of a step (prep, qkv, o, gu, down)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ms_chain -s 1 -c 4 -o gpurun_out/s3_chain_layer python bench.py --batch 8 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_chain_layer.log 2>&1; echo "ncu exit $?"
