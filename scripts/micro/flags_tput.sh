# block_tput under different ptxas settings (diagnostics)
set -e
for f in "" "-Xptxas --allow-expensive-optimizations=true" "-maxrregcount=128" "-maxrregcount=80"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude $f -o /tmp/btf scripts/micro/block_tput.cu
  echo "flags: ${f:-default}"; /tmp/btf | grep -E "bs=1 links=1 head=0 threads 256 x 2|bs=1 links=1 head=1"
done
