# ncu evidence for one round (argument: round tag, default r2) -> gpurun_out/
#  1. launch list of two steps with per-launch DRAM bytes (the HBM side of the tails)
#  2. one full-set capture (source-level) of the tensor-core kernels of one step
TAG=${1:-r2}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python tools/profile_step.py --steps 2 > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"logits_kernel|gemm_kernel" -c 2 \
    -o gpurun_out/prof_${TAG} -f python tools/profile_step.py --steps 1 > gpurun_out/prof_${TAG}.log 2>&1
