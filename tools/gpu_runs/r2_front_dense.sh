# dense first layer (C = 1 + pool): front tests, model tests, front time
timeout 600 python -m pytest -x -q tests/test_gpu_front.py 2>&1 | tail -3
for a in fashion cifar10; do timeout 120 python tools/front_time.py --arch $a --batch 65536; done
timeout 900 python -m pytest -x -q tests/test_gpu_model.py tests/test_gpu_net.py 2>&1 | tail -2
