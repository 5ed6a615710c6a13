# ncu captures of the C3 (mPSO + NR) kernels
O=${OUT:-gpurun_out/prof_c3}; mkdir -p $O
python tools/profile_case.py c3 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python tools/profile_case.py c3 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"pso_walk|refine_strip|tc_surface|bfs_tc_kernel" -s 4 -c 4 -o $O/c3 python tools/profile_case.py c3 2 > $O/c3.log 2>&1
ls $O
