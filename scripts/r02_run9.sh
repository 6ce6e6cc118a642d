timeout 600 python bench.py 2>&1 | tail -2
YCHG_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --size 8192 --steps 4 --warmup 2 2>&1 | tail -4
YCHG_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --size 8192 --steps 4 --warmup 2 --pattern random 2>&1 | tail -4
timeout 300 python bench.py --impl reference 2>&1 | tail -2
