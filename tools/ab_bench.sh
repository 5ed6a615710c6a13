# A/B the in-tree library against tools/var/lib_*.so on one config (stage averages).
cfg=${1:-c5}
for lib in paper_1905_06228_b200/libdicb200.so tools/var/lib_*.so; do
  for dxc in ${DXCS:-""}; do :; done
  DICB200_LIB=$PWD/$lib CONFIGS=$cfg bash tools/quick_bench.sh | sed "s|^|$(basename $lib) |"
done
