# hot-loop rate with parts removed (diagnostics): full lean block, K3 only, K1 only
set -e
for v in "" "-DYCHG_DIAG_NO_K1"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude $v -o /tmp/bt$v scripts/micro/block_tput.cu
  echo "variant: ${v:-full}"; /tmp/bt$v
done
