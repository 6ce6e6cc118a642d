# Round profile capture (1 GPU): plain run, launch list, full ncu set on the scan
# and finish kernels, and the launch list of one device decomposition.
set -e
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/prof_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ychg_scan_kernel -s 4 -c 1 -o gpurun_out/prof_scan $B > gpurun_out/prof_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ychg_finish_kernel -s 4 -c 1 -o gpurun_out/prof_finish $B > gpurun_out/prof_full2.log 2>&1
D="python -c 'import paper_1307_2560_b200 as y; img=y.synth(\"checker\",21000,21000,cell=7); y.decompose(img); print(y.decompose(img).edge_count)'"
eval $D > gpurun_out/prof_dec_plain.log 2>&1
eval ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/dec_launches.csv $D > gpurun_out/prof_dec.log 2>&1
echo done
