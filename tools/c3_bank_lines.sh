O=gpurun_out/c3src
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for K in k_ws_sort k_mod0_window k_ps_refine k_nx_emit k_merge_tile_rec k_ws_part1 k_ws_part2 k_ws_count k_nx_window; do
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$K -c 1 -o $O/$K python tools/profile_once.py 268435456 > $O/ncu_$K.log 2>&1
  python tools/ncu_lines_col.py $O/$K.ncu-rep "L1 Wavefronts Shared Excessive" 12 > $O/$K.excess.txt 2>&1
  rm -f $O/$K.ncu-rep
done
