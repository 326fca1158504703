#!/bin/bash
# One gpurun session: GPU tests, bench lines, ncu launch list + one full capture.
# usage: tools/gpu_check.sh TAG [tests] [bench] [ncu]
TAG=${1:-x}; shift
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
for what in "$@"; do
  case $what in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; tail -3 $O/tests.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log ;;
    c2|c3|c4|c5|store|fasta|cartesian) timeout 900 python bench.py --workload $what > $O/bench_$what.json 2> $O/bench_$what.err; tail -c 600 $O/bench_$what.json; tail -3 $O/bench_$what.err ;;
    ref) timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; cat $O/bench_ref.json ;;
    ncu_c2) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file $O/c2_launches.csv python tools/profile_once.py c2 > $O/ncu_c2.log 2>&1; python tools/ncu_summary.py $O/c2_launches.csv > $O/c2_launches.txt; head -30 $O/c2_launches.txt ;;
    ncu_c4|ncu_c5) W=${what#ncu_}; timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file $O/${W}_launches.csv python tools/profile_once.py $W > $O/ncu_$W.log 2>&1; python tools/ncu_summary.py $O/${W}_launches.csv 40 > $O/${W}_launches.txt; head -25 $O/${W}_launches.txt ;;
    ncu_c3) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file $O/c3_launches.csv python tools/profile_once.py 268435456 > $O/ncu_c3.log 2>&1; python tools/ncu_summary.py $O/c3_launches.csv > $O/c3_launches.txt; head -30 $O/c3_launches.txt ;;
    c3full_*) K=${what#c3full_}; timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$K -c 1 -o $O/c3full_$K python tools/profile_once.py 268435456 > $O/ncu_c3full_$K.log 2>&1; tail -2 $O/ncu_c3full_$K.log ;;
    c5full_*) K=${what#c5full_}; timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$K -c 1 -o $O/c5full_$K python tools/profile_once.py c5 > $O/ncu_c5full_$K.log 2>&1; tail -2 $O/ncu_c5full_$K.log ;;
    c4full_*) K=${what#c4full_}; timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$K -c 1 -o $O/c4full_$K python tools/profile_once.py c4 > $O/ncu_c4full_$K.log 2>&1; tail -2 $O/ncu_c4full_$K.log ;;
    c2full_*) K=${what#c2full_}; timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$K -c 1 -o $O/c2full_$K python tools/profile_once.py c2 > $O/ncu_c2full_$K.log 2>&1; tail -2 $O/ncu_c2full_$K.log ;;
    full_*) K=${what#full_}; timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$K -c 1 -o $O/full_$K python tools/profile_once.py c2 > $O/ncu_full_$K.log 2>&1; tail -3 $O/ncu_full_$K.log ;;
  esac
done
# extra: full ncu capture of one launch of kernel K on the C3-size run: tools/gpu_check.sh TAG c3full_K
# c4full_K: full ncu capture of one launch of kernel K in one C4 wave
# store: .saix pack / crc / unpack timing at 2^27
for what in "$@"; do
  case $what in
    store) timeout 600 python tools/store_probe.py $((1<<27)) > $O/store.json 2> $O/store.err; cat $O/store.json; tail -3 $O/store.err ;;
    storetests) timeout 900 python -m pytest tests/test_gpu_index_store.py -x -q > $O/storetests.log 2>&1; tail -15 $O/storetests.log ;;
    ncu_store) timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/store_launches.csv python tools/store_probe.py $((1<<26)) > $O/ncu_store.log 2>&1; python tools/ncu_summary.py $O/store_launches.csv 20 > $O/store_launches.txt; head -20 $O/store_launches.txt ;;
  esac
done
for what in "$@"; do
  case $what in
    storefull_*) K=${what#storefull_}; timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -c 2 -o $O/storefull_$K python tools/store_probe.py $((1<<26)) > $O/ncu_storefull_$K.log 2>&1; tail -2 $O/ncu_storefull_$K.log ;;
  esac
done
for what in "$@"; do
  case $what in
    fastatests) timeout 900 python -m pytest tests/test_gpu_fasta.py -x -q > $O/fastatests.log 2>&1; tail -15 $O/fastatests.log ;;
  esac
done
for what in "$@"; do
  case $what in
    fastafull_*) K=${what#fastafull_}; timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -c 1 -o $O/fastafull_$K python bench.py --workload fasta --steps 3 --warmup 3 --no-cpu-baseline --no-prof > $O/ncu_fastafull_$K.log 2>&1; tail -2 $O/ncu_fastafull_$K.log ;;
  esac
done
for what in "$@"; do
  case $what in
    carttests) timeout 900 python -m pytest tests/test_gpu_cartesian.py -x -q > $O/carttests.log 2>&1; tail -25 $O/carttests.log ;;
  esac
done
for what in "$@"; do
  case $what in
    ncu_cart) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_ct_|k_pm1|k_sparse|k_scan" --csv --log-file $O/cart_launches.csv python bench.py --workload cartesian --steps 1 --warmup 3 --no-cpu-baseline --no-prof > $O/ncu_cart.log 2>&1; python tools/ncu_summary.py $O/cart_launches.csv 20 > $O/cart_launches.txt; head -20 $O/cart_launches.txt ;;
  esac
done
for what in "$@"; do
  case $what in
    cartfull_*) K=${what#cartfull_}; timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -c 1 -o $O/cartfull_$K python bench.py --workload cartesian --steps 1 --warmup 3 --no-cpu-baseline --no-prof > $O/ncu_cartfull_$K.log 2>&1; tail -2 $O/ncu_cartfull_$K.log ;;
  esac
done
for what in "$@"; do
  case $what in
    ncu_fasta) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_fa_|k_scan" --csv --log-file $O/fasta_launches.csv python bench.py --workload fasta --steps 1 --warmup 3 --no-cpu-baseline --no-prof > $O/ncu_fasta.log 2>&1; python tools/ncu_summary.py $O/fasta_launches.csv 20 > $O/fasta_launches.txt; head -12 $O/fasta_launches.txt ;;
    ncu_store2) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_crc|k_unpack|k_put|k_ps_|k_pairs" --csv --log-file $O/store_launches.csv python bench.py --workload store --steps 1 --warmup 3 --no-cpu-baseline --no-prof > $O/ncu_store.log 2>&1; python tools/ncu_summary.py $O/store_launches.csv 20 > $O/store_launches.txt; head -12 $O/store_launches.txt ;;
  esac
done
for what in "$@"; do
  case $what in
    c2nowin) SAIX_WINDOW_NAMING=0 timeout 900 python bench.py --workload c2 --no-cpu-baseline > $O/bench_c2nowin.json 2> $O/bench_c2nowin.err; tail -c 300 $O/bench_c2nowin.json ;;
    largetests) timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py tests/test_gpu_batch.py -x -q > $O/largetests.log 2>&1; tail -15 $O/largetests.log ;;
    sanitize) for tool in memcheck racecheck synccheck; do SAIX_WS_MIN_M=4096 timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 30 --kernel-name kns=k_ python tools/sanitize_run.py > $O/san_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|all steps|MISMATCH" $O/san_$tool.log | tail -3; done ;;
    traces) for w in c2 c3; do SAIX_TRACE=1 timeout 600 python tools/profile_once.py $( [ $w = c3 ] && echo 268435456 || echo c2 ) 2>&1 | grep "saix dc3" | sort | uniq -c > $O/trace_$w.txt; cat $O/trace_$w.txt; done ;;
  esac
done
