cfg=${1:-c4}
python tools/profile_case.py $cfg 1 > /dev/null || exit 1
ncu --set full --import-source on --clock-control none -k regex:refine_strip -c 1 -o gpurun_out/ref_full_$cfg python tools/profile_case.py $cfg 1 > gpurun_out/ref_full_$cfg.log 2>&1
