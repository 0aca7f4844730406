# final round-2 pass on the shipped build: tests, smoke, default bench, reference arm, 2-rank shared-GPU lines
set -x
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 -rfE 2>&1 | tail -30 > gpurun_out/fin_tests.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/fin_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
for P in 1 0; do
DISCO_PEER=$P DISCO_BENCH_SHARE_GPU=1 timeout 600 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$P bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/fin_share_peer$P.json 2>&1
done
