# A/B of the tensor-core conversions (flag 32768) on the other workloads
for w in "mnist3 21568" "cifar 24576"; do set -- $w
  for v in $2 $(( $2 | 32768 )); do HCNN_NTT_VARIANT=$v timeout 300 python bench.py --workload $1 --channels 1 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$1', $v, d['ms_per_step'], {n: round(x['ms_total'],3) for n,x in k.items() if 'scale' in n or 'extend' in n})"; done; done
