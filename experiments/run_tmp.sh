OUT=gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py -q -x > $OUT/t3.log 2>&1; tail -3 $OUT/t3.log
QVB_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --sample-seeds 0 > $OUT/bench2.json 2> $OUT/bench2.err
tail -5 $OUT/bench2.err
