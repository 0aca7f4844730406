# quick correctness pass after a kernel change: dual + parity + acceptance tests
timeout 1500 python -m pytest tests/test_gpu_dual.py tests/test_gpu_parity.py tests/test_gpu_acceptance.py -q --timeout 900 -rfE ${@} 2>&1 | tail -30 > gpurun_out/quick_tests.txt
