# Full ncu captures (--set full) of the top kernels, summarised on the box (reps deleted):
# tools/full_captures.sh; outputs in gpurun_out/s5f
set -x
O=gpurun_out/s5f
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_batch.py -x -q -m gpu -k ramped > $O/ramp_test.txt 2>&1
for K in k_ws_sort k_lcp_direct_p2 k_merge_tile_rec k_ps_refine k_nx_emit k_nx_window k_mod0_window k_ws_part1 k_ws_part2 k_ws_count; do
  bash tools/gpu_check.sh s5f c3full_$K > /dev/null 2>&1
done
bash tools/gpu_check.sh s5f c4full_k_pair_dc3 c5full_k_sparse_query > /dev/null 2>&1
python tools/full_summary.py $O/*.ncu-rep > $O/full_summaries.txt 2>&1
for r in $O/*.ncu-rep; do b=$(basename $r .ncu-rep); python tools/ncu_lines.py $r 1 40 > $O/$b.lines.txt 2>&1; done
rm -f $O/*.ncu-rep
ls $O
