#!/bin/bash
OUT=gpurun_out; T=r02m; mkdir -p $OUT
timeout 900 python experiments/r02/upload_trace.py > $OUT/${T}_upload.txt 2>&1; cat $OUT/${T}_upload.txt
