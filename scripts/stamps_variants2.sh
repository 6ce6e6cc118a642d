for cfg in "libychg_b200.so 8" "libychg_b200_w8s4_compute_only.so 8" "libychg_b200_w16s2_compute_only.so 16" "libychg_b200_w8s4_no_head.so 8" "libychg_b200_w12s3.so 12" "libychg_b200_w16s2.so 16"; do
  set -- $cfg
  for pat in hbands random; do
    echo "== $1 $pat"; YCHG_LIB=paper_1307_2560_b200/$1 python scripts/stamps.py 21000 $pat full $2 2>&1 | grep -E 'warp done|merged|exit'
  done
done
