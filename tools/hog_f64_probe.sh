timeout 600 python -m pytest tests/test_sgd_gpu.py -x -q --timeout 300 2>&1 | tail -2
for v in b3 b4 b2 r16; do
  NOMAD_B200_LIB=$PWD/paper_2505_15511_b200/variants/$v.so timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --knn-mode bf16 > gpurun_out/var_$v.json 2>gpurun_out/var_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/var_$v.json').read().strip().splitlines()[-1]);print('$v f64', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), round(d['value']/1e9,1), 'G/s | df', round(d['double_float_rows']['ms_per_step'],3), round(d['double_float_rows']['value']/1e9,1), 'frac', round(d['double_float_rows']['roofline']['frac'],3))" || tail -3 gpurun_out/var_$v.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sgd_hogwild -s 2 -c 1 -o gpurun_out/sgd_f64 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --knn-mode bf16 > gpurun_out/ncu_sgd_f64.log 2>&1; tail -1 gpurun_out/ncu_sgd_f64.log
