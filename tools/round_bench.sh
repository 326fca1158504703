#!/bin/bash
# Round-end measurement set (one gpurun call): default bench line (C4 + C3
# block), the reference arm, C5 and C2 lines, smoke.  usage: tools/round_bench.sh TAG
T=${1:-s2n}
O=gpurun_out/$T
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for w in c5 c2; do timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
tail -c 400 $O/bench_default.json; echo; cat $O/bench_reference.json | head -c 300; echo; tail -1 $O/smoke.log
