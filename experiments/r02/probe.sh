set -x
free -g; nproc; lscpu | grep -i "model name\|socket\|numa"; nvidia-smi --query-gpu=name,memory.total --format=csv
ulimit -a | head -5
( time python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline ) > gpurun_out/r02a_c4_e2e.json 2> gpurun_out/r02a_c4_e2e.err
tail -5 gpurun_out/r02a_c4_e2e.err
