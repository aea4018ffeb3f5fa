#!/bin/bash
# r02ar: C5 gather sweeps on the final code for the C3 (602-dim rows) and C2 (100-dim) graphs
OUT=gpurun_out; T=r02ar; mkdir -p $OUT
timeout 1200 python experiments/gather_sweep.py C3 > $OUT/${T}_gather_sweep_C3.jsonl 2> $OUT/${T}_gather_sweep_C3.err; echo C3 rc=$?
timeout 1200 python experiments/gather_sweep.py C2 > $OUT/${T}_gather_sweep_C2.jsonl 2> $OUT/${T}_gather_sweep_C2.err; echo C2 rc=$?
