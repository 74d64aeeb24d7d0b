# scaled-net conv2 passes (configs[4] shapes, 1 GPU): wgrad unit order / accumulation-split variants,
# timed alone (pass_bench) and one ncu --set full capture of the wgrad kernel per variant
A="--B 256 --H 110 --K1 512 --K2 2048 --reps 2"
for v in "CP_TC_WGRAD_ORDER=0" "CP_TC_WGRAD_ORDER=1" "CP_TC_WGRAD_ORDER=1 CP_TC_ACC_TERMS=1073741824"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 120 python scripts/pass_bench.py $A > gpurun_out/pb_$tag.json 2>&1
  env $v timeout 600 ncu --set full --clock-control none -k regex:conv_tc_kernel --kernel-name-base demangled \
      --launch-skip 1 -c 1 -o gpurun_out/sc_wgrad_$tag python scripts/pass_bench.py --B 256 --H 110 --K1 512 \
      --K2 2048 --reps 1 > gpurun_out/ncu_$tag.log 2>&1
done
