set -e
cd /root/repo
mkdir -p build/stats
for f in paper_2510_03312_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude -DUBS_FWD_STATS -c $f -o build/stats/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o profiles/tools/libubs_stats.so build/stats/*.o -lcudart
