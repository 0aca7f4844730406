timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-exchange-leg --no-cpu-baseline > gpurun_out/lds_bench.json 2> gpurun_out/lds_bench.err
bash tools/gpu_prof.sh r2
