# A/B of the products kernel at C4 + bit-exactness tests of the segmented paths
OUT=gpurun_out; T=${1:-r02b}
python -m pytest tests/test_access_prob_gpu.py -q -x -k "segmented or node_major or c4 or first_sweep" > $OUT/${T}_aptests.log 2>&1; tail -3 $OUT/${T}_aptests.log
B="python bench.py --config C4 --no-cpu-baseline --no-e2e --sample-seeds 0 --steps 10 --warmup 3"
QVB_PRODUCTS=lockstep $B > $OUT/${T}_c4_lockstep.json 2>$OUT/${T}_c4_lockstep.err
$B > $OUT/${T}_c4_tma.json 2>$OUT/${T}_c4_tma.err

for t in lockstep tma; do python -c "
import json,sys;d=json.load(open('$OUT/${T}_c4_'+sys.argv[1]+'.json'));a=d['access_prob'];print(sys.argv[1],a['ms_per_call'],a['survey_model']['frac'],{k:round(v['ms_per_call'],3) for k,v in a['kernels'].items()})" $t; done
ncu --set full --clock-control none --import-source on -k regex:k_products -s 2 -c 1 -o $OUT/${T}_products -f $B --steps 3 > /dev/null 2>&1; echo ncu=$?
