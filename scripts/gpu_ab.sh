for i in 1 2; do
for v in libif_head libif_b200; do
IFB_LIB_PATH=/root/repo/paper_2401_08294_b200/$v.so python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"
done; done
