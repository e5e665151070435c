timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "sgd or hogwild or quality or trainer or fit or smoke" 2>&1 | tail -3
for v in g4b3f64 g4b3df g8b3df g4b4df; do
  NOMAD_B200_LIB=$PWD/paper_2505_15511_b200/variants/$v.so timeout 200 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/var_$v.json 2>gpurun_out/var_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/var_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), round(d['value']/1e9,1), 'G/s loss', round(d['config']['final_loss'],4))" || tail -3 gpurun_out/var_$v.err
done
for v in g4b3f64 g4b3df; do
  for cfg in "20000 32 10 200" "200000 64 20 100"; do
    echo $v $cfg; NOMAD_B200_LIB=$PWD/paper_2505_15511_b200/variants/$v.so timeout 300 python tools/hog_quality.py $cfg
  done
done
