# stream-tail finishing kernels: 8-piece load batches (new) vs 4 / 1 (old), ncu durations; parity
for v in old new; do for P in 1 4 8; do
  CP_LIB=exp/libconvpart_tail$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tail --csv \
    --log-file gpurun_out/r02t_${v}_P$P.csv python scripts/pass_bench.py --P $P --reps 3 > gpurun_out/r02t_${v}_P$P.log 2>&1; echo "$v P=$P rc=$?"
done; done
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_trajectory.py tests/test_gpu_full_size.py -x -q -m gpu > gpurun_out/r02t_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02t_tests.log
