#!/bin/bash
# r01h: round evidence — full GPU tests, bench lines (C2 default, C4, C3, host tier, reference),
# launch lists and ncu captures of the dominant kernels
OUT=gpurun_out; TAG=r01h
mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu > $OUT/${TAG}_tests.log 2>&1; tail -2 $OUT/${TAG}_tests.log
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
timeout 600 python bench.py --impl reference > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err
timeout 900 python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 10 > $OUT/${TAG}_bench_c4.json 2> $OUT/${TAG}_bench_c4.err
timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 10 --batch 262144 > $OUT/${TAG}_bench_c3.json 2> $OUT/${TAG}_bench_c3.err
timeout 600 python bench.py --host-frac 0.25 --no-cpu-baseline --no-e2e --steps 10 > $OUT/${TAG}_bench_host25.json 2> $OUT/${TAG}_bench_host25.err
QVB_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --sample-seeds 0 > $OUT/${TAG}_bench_2rank_1gpu.json 2> $OUT/${TAG}_bench_2rank_1gpu.err
B="python bench.py --steps 3 --warmup 3 --clock-window 0 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/${TAG}_launches_c4.csv $B --config C4 --sample-seeds 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_codes" -s 7 -c 7 -o $OUT/${TAG}_c4_codes -f python experiments/ap_bench.py C4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather -s 3 -c 1 -o $OUT/${TAG}_gather -f $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_first -s 1 -c 1 -o $OUT/${TAG}_c2_first -f $B > /dev/null 2>&1
echo done
