# unpool: four pooled rows' loads in flight per thread (unp4) vs one (unp1); ncu at P=1 / 4, slice steps, parity
for v in unp1 unp4; do for P in 1 4; do
  CP_LIB=exp/libconvpart_$v.so P=$P STEPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"unpool|bias_grad" --csv --log-file gpurun_out/r02u_${v}_P$P.csv python scripts/slice_step.py > /dev/null 2>&1; echo "$v P=$P rc=$?"
  CP_LIB=exp/libconvpart_$v.so P=$P timeout 300 python scripts/slice_step.py > gpurun_out/r02u_${v}_P$P.json 2>&1; tail -1 gpurun_out/r02u_${v}_P$P.json
done; done
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_trajectory.py tests/test_gpu_full_size.py tests/test_gpu_loopback.py tests/test_gpu_probe_tiny.py -x -q -m gpu > gpurun_out/r02u_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02u_tests.log
