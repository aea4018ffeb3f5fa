OUT=gpurun_out
for m in 0 1 2 3; do QVB_G_STORE=$m timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_sector_op_read_hit_rate.pct --clock-control none --csv -k regex:"k_codes" --log-file $OUT/kc_s$m.csv python experiments/ap_bench.py C4 > /dev/null 2>&1; done
