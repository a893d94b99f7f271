timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_front.py tests/test_gpu_layers.py -x -q -m gpu > gpurun_out/pitch1_tests.log 2>&1; tail -2 gpurun_out/pitch1_tests.log
timeout 300 python tools/determinism.py --reps 10 --batch 262144 --plan '{"2": [1, 0, 6]}'
timeout 900 python bench.py --steps 5 --warmup 3 --no-extra --no-cpu > gpurun_out/pitch1_bench.json 2> gpurun_out/pitch1_bench.err
python3 -c "import json; d=json.load(open('gpurun_out/pitch1_bench.json')); print(d['value'], d['e2e']['value'], d['clocks'], d['throughput_plan']['variants'], {k: v['ms'] for k, v in d['roofline']['per_op'].items()})"
