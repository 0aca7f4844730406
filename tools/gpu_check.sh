set -x
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -40 > gpurun_out/gpu_tests_r2a.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1_r2a.json 2> gpurun_out/bench_n1_r2a.err
for P in 1 0; do
DISCO_PEER=$P DISCO_BENCH_SHARE_GPU=1 timeout 600 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$P bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench_share_peer$P.json 2>&1
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r2a.json 2>&1
