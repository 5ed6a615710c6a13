# Build libdicb200 variants differing only in bfs_bs.cu compile flags (A/B on the GPU via DICB200_LIB).
set -e
cd /root/repo
mkdir -p tools/var
B=paper_1905_06228_b200/build
objs=$(ls $B/*.o | grep -v bfs_bs.cu.o)
for v in "$@"; do
  name=$(echo "$v" | tr -c 'A-Za-z0-9' '_')
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -I include -I paper_1905_06228_b200/csrc $v -c paper_1905_06228_b200/csrc/bfs_bs.cu -o /tmp/bs_$name.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/var/lib_$name.so $objs /tmp/bs_$name.o -lpthread
  echo tools/var/lib_$name.so
done
