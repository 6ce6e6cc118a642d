# Round profile capture (1 GPU): plain run, launch list, full ncu set on the scan kernel.
set -e
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/prof_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ychg_scan_kernel -s 4 -c 1 -o gpurun_out/prof_scan $B > gpurun_out/prof_full.log 2>&1
echo done
