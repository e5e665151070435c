# Per-config measurements with the reference CPU epoch beside
for cfg in A B C8 C; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 2>/dev/null | tail -1 > gpurun_out/cfg_$cfg.json
  timeout 900 python bench.py --config $cfg --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 > gpurun_out/cfg_${cfg}_ref.json
done
