# pageable host path: copy threads x staging chunk size (scripts/pageable_probe.py)
T=${T:-"4 8 16"}; MB=${MB:-"2 4 8 16"}
for rep in 1 2; do for t in $T; do for mb in $MB; do
  echo -n "threads=$t chunk=${mb}MB: "; YCHG_COPY_THREADS=$t YCHG_STAGE_MB=$mb python scripts/pageable_probe.py 2>&1 | grep "^pageable"
done; done; done
