# ncu --set full of the chain's gate/up kernel (launch 4 of the step: prep, qkv, o, gu), B = 8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ms_chain -s 3 -c 1 -o gpurun_out/s3_chain_gu python bench.py --batch 8 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_chain.log 2>&1; echo "ncu exit $?"
