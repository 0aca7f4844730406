# round-2 evidence pass: bench (N=1), smoke, all -m gpu tests, ncu launch list + full capture, 2-rank shared-GPU bench both transports, reference arm
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2f_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r2f_smoke.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 -rfE 2>&1 | tail -60 > gpurun_out/r2f_tests.txt
bash tools/gpu_prof.sh r2f
for P in 1 0; do
DISCO_PEER=$P DISCO_BENCH_SHARE_GPU=1 timeout 600 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$P bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/r2f_share_peer$P.json 2>&1
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2f_ref.json 2> gpurun_out/r2f_ref.err
