#!/bin/bash
# Round-end validation in one gpurun call: full GPU tests, the
# bench set (default / reference / c5 / c2 / smoke) and a 2-rank run.
# usage: tools/final_check.sh TAG
T=${1:-s6}
O=gpurun_out/$T
mkdir -p $O
bash tools/gpu_check.sh $T tests > $O/check.log 2>&1
tail -3 $O/tests.log
cat $O/check.log | grep -E "rc=|SUMMARY"
bash tools/round_bench.sh $T
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_gpus2.json 2> $O/bench_gpus2.err
tail -c 300 $O/bench_gpus2.json
