timeout 600 python -m pytest tests/test_sgd_gpu.py -x -q --timeout 300 2>&1 | tail -3
for v in base late3 late4; do
  NOMAD_B200_LIB=$PWD/paper_2505_15511_b200/variants/$v.so timeout 200 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --knn-mode bf16 > gpurun_out/var_$v.json 2>gpurun_out/var_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/var_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), round(d['value']/1e9,1), 'G/s loss', round(d['config']['final_loss'],4))" || tail -3 gpurun_out/var_$v.err
done
