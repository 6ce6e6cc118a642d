# Round-2 profile capture (1 GPU): plain bench, launch list, ncu --set full of one
# scan launch, graph-level ncu of the K=20 scan graph, decompose/profile launches.
set -x
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
$B > gpurun_out/p2_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/p2_launches.csv $B > gpurun_out/p2_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ychg_scan_kernel -s 10 -c 1 -o gpurun_out/p2_scan python scripts/graph_profile.py 20 hbands > gpurun_out/p2_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ychg_scan_kernel -s 10 -c 1 -o gpurun_out/p2_scan_random python scripts/graph_profile.py 20 random > gpurun_out/p2_full_r.log 2>&1
ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/p2_graph.csv python scripts/graph_profile.py 20 hbands > gpurun_out/p2_graph.log 2>&1
ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/p2_graph_random.csv python scripts/graph_profile.py 20 random > gpurun_out/p2_graph_r.log 2>&1
echo done
