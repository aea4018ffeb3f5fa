#!/bin/bash
# r02ao: final check after the fused-pass experiment: GPU suite, smoke, default bench line
OUT=gpurun_out; T=r02ao; mkdir -p $OUT
timeout 2400 python -m pytest tests -q -m gpu > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${T}_smoke.log 2>&1; tail -1 $OUT/${T}_smoke.log
timeout 1700 python bench.py --steps 20 --warmup 5 > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
python -c "
import json; d=json.load(open('$OUT/${T}_bench.json')); a=d['access_prob']
print('gather', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['frac_of_d2h_ceiling'],3), 'P', round(a['ms_per_call'],3), round(a['survey_model']['frac'],4), 'bitident', a['cpu_baseline'].get('bit_identical_nodes'), d['clocks'])"
