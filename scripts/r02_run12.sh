for pat in random hbands; do
  YCHG_LIB=paper_1307_2560_b200/libychg_b200_r1.so timeout 120 python scripts/ab_graph.py 21000 $pat
  for k in "" 4 3 2; do YCHG_SEGMENTS=$k timeout 120 python scripts/ab_graph.py 21000 $pat; done
done
