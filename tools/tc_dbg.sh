for d in ${DBGS:-0 1 2 3}; do
  DICB200_TC_DBG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bfs_tc_kernel --csv python tools/profile_case.py ${1:-c5} 1 2>/dev/null | grep bfs_tc | awk -F'","' -v d=$d '{print "dbg", d, $NF}'
done
