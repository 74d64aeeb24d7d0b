# ncu --set full of the conv2 GEMMs at the P=4 and P=8 slice shapes (1 GPU, LOCAL mode, pass_bench)
for P in 4 8; do
timeout 300 python scripts/pass_bench.py --P $P --reps 2 > gpurun_out/r02k_plain_p$P.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -c 6 -o gpurun_out/r02k_p$P python scripts/pass_bench.py --P $P --reps 1 > gpurun_out/r02k_ncu_p$P.log 2>&1; echo "P=$P ncu rc=$?"
done
