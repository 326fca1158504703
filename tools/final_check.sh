O=gpurun_out/s6
mkdir -p $O
bash tools/gpu_check.sh s6 tests > /dev/null 2>&1
tail -3 $O/tests.log
bash tools/round_bench.sh s6
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_gpus2.json 2> $O/bench_gpus2.err
tail -c 600 $O/bench_gpus2.json
