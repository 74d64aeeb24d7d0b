# ncu --set full of the head kernels at P=1 and P=4 (one rank's compute-only step)
for P in 1 4; do
P=$P STEPS=2 timeout 600 ncu --set full --clock-control none -k regex:"fc_fwd_partial|fc_bwd_cols|fc_fwd_reduce|unpool_kernel" -c 4 -o gpurun_out/r02fc_P$P python scripts/slice_step.py > gpurun_out/r02fc_P$P.log 2>&1; echo "P=$P rc=$?"
done
