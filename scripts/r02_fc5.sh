# fc_fwd_partial: 5 CTAs per SM (launch bounds + max shared carveout) vs 4 (1.01 waves at P=1)
for v in fc4 fc5; do for P in 1 4; do
  CP_LIB=exp/libconvpart_$v.so P=$P STEPS=3 timeout 300 ncu --metrics gpu__time_duration.sum,launch__waves_per_multiprocessor --clock-control none -k regex:"fc_fwd_partial" --csv --log-file gpurun_out/r02g_${v}_P$P.csv python scripts/slice_step.py > /dev/null 2>&1; echo "$v P=$P rc=$?"
  CP_LIB=exp/libconvpart_$v.so P=$P timeout 300 python scripts/slice_step.py > gpurun_out/r02g_${v}_P$P.json 2>&1; tail -1 gpurun_out/r02g_${v}_P$P.json
done; done
timeout 900 python -m pytest tests/test_gpu_layers.py -x -q -m gpu -k "head or full_step" > gpurun_out/r02g_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02g_tests.log
