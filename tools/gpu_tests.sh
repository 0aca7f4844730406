# GPU test pass (gpurun): all -m gpu tests, per-test timeout, log under gpurun_out/
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -rfE ${@} 2>&1 | tail -60 > gpurun_out/gpu_tests.txt
