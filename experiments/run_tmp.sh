OUT=gpurun_out
for cfg in "QVB_SEG0_MB=32" "QVB_SEG0_MB=48" "QVB_SEG0_MB=48 QVB_SEG_MB=72" "QVB_SEG0_MB=56 QVB_SEG_MB=72" "QVB_SEG0_MB=40 QVB_SEG_MB=80"; do echo "$cfg" >> $OUT/ap5.log; env $cfg timeout 300 python experiments/ap_bench.py C4 >> $OUT/ap5.log 2>&1; done
