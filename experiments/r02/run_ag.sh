#!/bin/bash
# r02ag: P-weighted ids at small host fractions: which host-list knob limits the class split
OUT=gpurun_out; T=r02ag; mkdir -p $OUT
timeout 1500 python experiments/r02/host_knobs.py --p-weighted --more > $OUT/${T}_host_knobs_pw.txt 2>&1; cat $OUT/${T}_host_knobs_pw.txt
