# why does the first bench.py of a fresh process tree sometimes print no JSON line?
( time timeout 300 python bench.py --scheme Q8_B64 --steps 50 --warmup 3 --no-cpu-baseline ) > gpurun_out/fb1.out 2> gpurun_out/fb1.err; echo "exit $?"
tail -c 600 gpurun_out/fb1.out; echo; tail -20 gpurun_out/fb1.err
( time timeout 300 python bench.py --scheme Q8_B64 --steps 50 --warmup 3 --no-cpu-baseline ) > gpurun_out/fb2.out 2> gpurun_out/fb2.err; echo "exit2 $?"; tail -c 300 gpurun_out/fb2.out; echo; tail -5 gpurun_out/fb2.err
