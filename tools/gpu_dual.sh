# quick GPU pass over the dual-backward work: new tests + parity, then a short bench
timeout 1500 python -m pytest tests/test_gpu_dual.py tests/test_gpu_parity.py -q --timeout 600 -rfE 2>&1 | tail -40 > gpurun_out/dual_tests.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/dual_smoke.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-fused > gpurun_out/dual_bench.json 2> gpurun_out/dual_bench.err
