# ncu capture of one step's tensor-core kernels (source-level, full set) -> gpurun_out/
ncu --set full --import-source on --clock-control none -k regex:"logits_kernel|gemm_kernel" -c 2 \
    -o gpurun_out/prof_${1:-r2} -f python tools/profile_step.py --steps 1 > gpurun_out/prof_${1:-r2}.log 2>&1
