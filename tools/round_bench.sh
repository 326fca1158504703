mkdir -p gpurun_out/s2n
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/s2n/bench_default.json 2> gpurun_out/s2n/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/s2n/bench_reference.json 2> gpurun_out/s2n/bench_reference.err
for w in c5 c2; do timeout 600 python bench.py --workload $w > gpurun_out/s2n/bench_$w.json 2> gpurun_out/s2n/bench_$w.err; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2n/smoke.log 2>&1
tail -c 400 gpurun_out/s2n/bench_default.json; echo; cat gpurun_out/s2n/bench_reference.json | head -c 300; echo; tail -1 gpurun_out/s2n/smoke.log
