# attention split-merge with batched loads: parity + KV decode bench + launch list at B=1
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_lm.py -q -x --timeout 600 > gpurun_out/attn_pytest.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/attn_pytest.log
for P in 255 1023; do for B in 1 8; do
  timeout 300 python bench.py --kv-pos $P --batch $B --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pos=$P B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms launches/step', d['gpu_launches']//d['steps'])"
done; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_mk|rope|attn" --launch-skip 200 -c 97 --csv --log-file gpurun_out/kv1_launches.csv python bench.py --kv-pos 255 --batch 1 --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu $?"
timeout 300 python scripts/engine_bench.py 2>&1 | tail -1 | cut -c1-200
