#!/bin/bash
# r02o: lookup cost in front of the row gather (L2-resident vs 888 MB table),
# host tier through cuMemCreate(HOST_NUMA) vs cudaHostAlloc, host NUMA layout
OUT=gpurun_out; T=r02o; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rgl experiments/r02/rowgather_lut.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hv experiments/r02/host_vmm.cu -lcuda
(lscpu | head -30; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c; numactl -H 2>/dev/null; nvidia-smi topo -m) > $OUT/${T}_host.txt 2>&1
timeout 600 /tmp/rgl > $OUT/${T}_rowgather_lut.txt 2>&1; cat $OUT/${T}_rowgather_lut.txt
timeout 900 /tmp/hv > $OUT/${T}_host_vmm.txt 2>&1; cat $OUT/${T}_host_vmm.txt
