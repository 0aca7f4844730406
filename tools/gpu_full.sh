# full GPU pass: every -m gpu test (no -x), smoke, 1-GPU bench; logs under gpurun_out/
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err
timeout 300 python __graft_entry__.py --smoke > gpurun_out/full_smoke.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 -rfE ${@} 2>&1 | tail -80 > gpurun_out/full_tests.txt
