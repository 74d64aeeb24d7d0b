# head kernels: shared-memory carveout for fc_fwd_partial (one wave at P=1), all-in-flight lane loads in
# fc_fwd_reduce / bias_grad_final; old vs new library, ncu durations at P=1 / 4, parity, N=1 bench
for v in fcold fcnew; do for P in 1 4; do
  CP_LIB=exp/libconvpart_$v.so P=$P STEPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fc_|bias_grad|softmax" --csv --log-file gpurun_out/r02f_${v}_P$P.csv python scripts/slice_step.py > /dev/null 2>&1; echo "$v P=$P rc=$?"
  CP_LIB=exp/libconvpart_$v.so P=$P timeout 300 python scripts/slice_step.py > gpurun_out/r02f_${v}_P$P.json 2>&1; tail -1 gpurun_out/r02f_${v}_P$P.json
done; done
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_trajectory.py tests/test_gpu_full_size.py tests/test_gpu_probe_tiny.py -x -q -m gpu > gpurun_out/r02f_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02f_tests.log
