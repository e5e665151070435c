# config D: kNN-graph build sweep 1M-10M x 768 (64 blobs, C = n/156250 >= 8), warm timings
for n in 1000000 2000000 5000000 10000000; do
  C=$(( n / 156250 )); [ $C -lt 8 ] && C=8
  for m in bf16 exact; do timeout 900 python tools/knn_time.py $n 768 $C $m; done
done
timeout 900 python tools/index_bench.py 5000000 768 32 --modes bf16,exact --recall | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('recall@15 bf16 vs exact at 5M:', d.get('recall_at_k'))"
