for k in 4 7; do YCHG_SEGMENTS=$k timeout 120 python scripts/ab_graph.py 21000 random; YCHG_NO_SKIP=1 YCHG_SEGMENTS=$k timeout 120 python scripts/ab_graph.py 21000 random; done
YCHG_SEGMENTS=4 YCHG_LIB=paper_1307_2560_b200/libychg_b200_w4s3_p_alu.so timeout 120 python scripts/ab_graph.py 21000 random
YCHG_SEGMENTS=4 YCHG_NO_SKIP=1 YCHG_LIB=paper_1307_2560_b200/libychg_b200_w4s3_p_alu.so timeout 120 python scripts/ab_graph.py 21000 random
