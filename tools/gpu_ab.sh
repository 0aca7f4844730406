# same-process A/B of the current build against abtmp/*.so builds (args: extra ab_kernels flags)
timeout 900 python tools/ab_kernels.py --so abtmp/*.so --reps 15 ${@} > gpurun_out/ab.txt 2>&1
