# config D: kNN-graph build sweep 1M-10M x 768, fp32-exact vs bf16 tcgen05 (C = n / 156250, 64 blobs)
for n in 1000000 2000000 5000000 10000000; do
  C=$(( n / 156250 )); [ $C -lt 8 ] && C=8
  timeout 900 python tools/index_bench.py $n 768 $C --modes bf16,exact --recall
done
