# Copy the judged summaries of a capture_round.sh output directory into
# profiles/ (tracked): bench lines, GPU test log, launch list + shares, ncu
# key metrics and per-line breakdowns. Usage: publish_capture.sh <capdir> <tag, e.g. r02>
set -e
C=$1; T=$2; P=${3:-profiles}
for c in c1 c2 c2b c3 c3x c4 c5; do
  [ -s $C/bench_$c.json ] && tail -1 $C/bench_$c.json > $P/${T}_bench_$c.json
done
[ -s $C/bench_ref_c5.json ] && tail -1 $C/bench_ref_c5.json > $P/${T}_bench_ref_c5.json
cp $C/pytest_gpu.txt $P/${T}_pytest_gpu.txt
grep '^"' $C/launches_bench_c5.csv > $P/${T}_ncu_launches_bench_c5.csv
python tools/launch_share.py $C/launches_bench_c5.csv > $P/${T}_launch_share_c5.txt
: > $P/${T}_ncu_summary.jsonl
[ -f $C/prof/refine.ncu-rep ] && python tools/summarize_ncu.py $C/prof/refine.ncu-rep refine_c5_steady >> $P/${T}_ncu_summary.jsonl
[ -f $C/prof/bs.ncu-rep ] && python tools/summarize_ncu.py $C/prof/bs.ncu-rep bs_ws_c5_steady >> $P/${T}_ncu_summary.jsonl
[ -f $C/prof/aux.ncu-rep ] && python tools/summarize_ncu.py $C/prof/aux.ncu-rep aux_c5_steady >> $P/${T}_ncu_summary.jsonl
[ -f $C/prof_c3/c3.ncu-rep ] && python tools/summarize_ncu.py $C/prof_c3/c3.ncu-rep c3 >> $P/${T}_ncu_summary.jsonl
[ -f $C/prof/refine.ncu-rep ] && python tools/ncu_src_top.py $C/prof/refine.ncu-rep refine.cu 40 > $P/${T}_ncu_lines_refine_c5.txt
[ -f $C/prof/bs.ncu-rep ] && python tools/ncu_src_top.py $C/prof/bs.ncu-rep bfs_bs.cu 40 > $P/${T}_ncu_lines_bs_ws_c5.txt
ls -la $P | grep ${T}_ | head -40
