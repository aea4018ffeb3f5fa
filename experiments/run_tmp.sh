OUT=gpurun_out
timeout 900 python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 20 --sample-seeds 0 > $OUT/b4.json 2> $OUT/b4.err
