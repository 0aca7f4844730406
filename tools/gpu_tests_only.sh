timeout 2000 python -m pytest tests -m gpu -q --timeout 900 -x -rfE 2>&1 | tail -40 > gpurun_out/gpu_tests_r2b.txt
