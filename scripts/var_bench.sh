for lib in libychg_b200.so "libychg_b200_w8s3_stages_links=2.so" "libychg_b200_w8s3_stages_links=2_warps_links=6.so" "libychg_b200_w8s3_stages_links=2_warps_links=8.so" "libychg_b200_w8s3_stages_links=4.so"; do
  for k in 100 20; do
    YCHG_LIB=$PWD/paper_1307_2560_b200/$lib python bench.py --steps $k --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$lib K=$k\", d[\"ms_per_step\"], d[\"north_star_subset\"][\"ms_per_step\"], d[\"config\"][\"plan\"])"
  done
done
