# functional check of bench.py's N-rank paths on ONE GPU (ranks share cuda:0, gloo plumbing)
export IFB_BENCH_SHARE_GPU=1
for cfg in "2 tensor" "2 layer" "4 hybrid"; do
  set -- $cfg
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $1 --steps 5 --warmup 3 --strategy $2 > gpurun_out/mr_$1_$2.json 2> gpurun_out/mr_$1_$2.err
  echo "$1 $2 rc=$? $(tail -c 400 gpurun_out/mr_$1_$2.json)"
  tail -2 gpurun_out/mr_$1_$2.err
done
