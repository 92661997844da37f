# tuning probe of the tensor-core conversions (tc_bconv.cuh): TMEM columns x CTAs per SM
for cc in "128 2" "128 4" "64 4" "64 6" "64 7"; do set -- $cc; HCNN_TC_COLS=$1 HCNN_TC_CTAS=$2 HCNN_NTT_VARIANT=57344 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$1 $2', d['ms_per_step'], k['k_extend_tc']['ms_total'], k['k_scale_tc']['ms_total'])"; done
