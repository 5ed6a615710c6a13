# steady-state (second pair of a fixed-first sequence) ncu captures of the C5 hot kernels
O=${OUT:-gpurun_out/prof}; mkdir -p $O
python tools/profile_seq.py c5 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine_strip -s 1 -c 1 -o $O/refine python tools/profile_seq.py c5 2 > $O/refine.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bs_ws_kernel -s 1 -c 1 -o $O/bs python tools/profile_seq.py c5 2 > $O/bs.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"bs_merge|bs_exact|tc_stats|bits_" -s 4 -c 5 -o $O/aux python tools/profile_seq.py c5 2 > $O/aux.log 2>&1
ls $O
