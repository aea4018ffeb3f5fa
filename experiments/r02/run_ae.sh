#!/bin/bash
# r02ae: PCIe copy-engine ceiling (the e2e bound); N=2 bench path on the final code (two ranks sharing the GPU)
OUT=gpurun_out; T=r02ae; mkdir -p $OUT
timeout 300 python experiments/r02/pcie_copy.py > $OUT/${T}_pcie_copy.txt 2>&1; cat $OUT/${T}_pcie_copy.txt
QVB_SHARE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config C2 --steps 5 --warmup 3 --no-cpu-baseline --sample-seeds 0 > $OUT/${T}_bench_n2.json 2> $OUT/${T}_bench_n2.err
echo rc=$?; tail -2 $OUT/${T}_bench_n2.err
python -c "
import json; d=json.load(open('$OUT/${T}_bench_n2.json')); a=d['access_prob']
print('n_gpus', d['n_gpus'], 'gather', d['value'], 'P', a['ms_per_call'], 'sharded', a.get('sharded_over_ranks'), d['placement']['fractions'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --config C1 --steps 3 --warmup 3 > $OUT/${T}_bench_ref_n2.json 2> $OUT/${T}_bench_ref_n2.err; echo refrc=$?; head -c 300 $OUT/${T}_bench_ref_n2.json
