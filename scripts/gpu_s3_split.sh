# chain: last-CTA split-K reduction; split-count sweep (IFB_MS_SPLITS=qkv,o,gu,down) at B=8
timeout 900 python -m pytest tests/test_gpu_stack.py -q -x --timeout 600 > gpurun_out/split_pytest.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/split_pytest.log
for sp in "" "3,8,1,8" "4,8,1,8" "4,8,2,8" "2,8,1,8" "4,6,1,6" "3,8,2,6"; do
IFB_MS_SPLITS=$sp timeout 300 python bench.py --batch 8 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/sp.log 2>&1; tail -1 gpurun_out/sp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splits=$sp', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"
done
python scripts/ms_timeline.py 8 3 2>&1 | tail -9
