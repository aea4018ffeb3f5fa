OUT=gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > $OUT/tall.log 2>&1; tail -2 $OUT/tall.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -2 $OUT/smoke.log
