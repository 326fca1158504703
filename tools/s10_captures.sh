#!/bin/bash
# Final-code ncu evidence (round 2, s10): launch lists of C3 / C4 / C5 and
# --set full captures of the C4 pair kernel, the C3 merge tile and window sort
# P3, summarised on the box.  usage: tools/s10_captures.sh
O=gpurun_out/s10
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
bash tools/gpu_check.sh s10 ncu_c4 ncu_c3 ncu_c5 > $O/lists.log 2>&1
bash tools/gpu_check.sh s10 c4full_k_pair_dc3 c3full_k_merge_tile_rec c3full_k_ws_sort > $O/full.log 2>&1
python tools/full_summary.py $O/*.ncu-rep > $O/full_summaries.txt 2>&1
for r in $O/*.ncu-rep; do b=$(basename $r .ncu-rep); python tools/ncu_lines.py $r 1 40 > $O/$b.lines.txt 2>&1; done
rm -f $O/*.ncu-rep $O/*.csv
ls $O
