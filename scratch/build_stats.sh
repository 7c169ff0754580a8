set -e
cd /root/repo
mkdir -p scratch/stats_build
for f in paper_2510_03312_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude -DUBS_FWD_STATS -c $f -o scratch/stats_build/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scratch/libubs_stats.so scratch/stats_build/*.o -lcudart
