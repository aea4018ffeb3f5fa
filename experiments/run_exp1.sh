OUT=gpurun_out
./experiments/l2_capacity > $OUT/exp1_l2cap.log 2>&1
for mb in 32 48 64 80 128; do echo "SEG_MB=$mb" >> $OUT/exp1_seg.log; QVB_SEG_MB=$mb timeout 300 python experiments/ap_bench.py C4 >> $OUT/exp1_seg.log 2>&1; done
