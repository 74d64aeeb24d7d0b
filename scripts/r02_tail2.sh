# stream-tail finishing kernels: one thread per pre-pool value, 16-piece load batches (new2) vs 8 (new) vs old
for v in old new new2; do for P in 1 4 8; do
  CP_LIB=exp/libconvpart_tail$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tail --csv \
    --log-file gpurun_out/r02t2_${v}_P$P.csv python scripts/pass_bench.py --P $P --reps 3 > gpurun_out/r02t2_${v}_P$P.log 2>&1; echo "$v P=$P rc=$?"
done; done
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_trajectory.py tests/test_gpu_full_size.py tests/test_gpu_loopback.py -x -q -m gpu > gpurun_out/r02t2_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02t2_tests.log
for rep in 1 2; do timeout 300 python bench.py > gpurun_out/r02t2_n1_$rep.json 2>/dev/null; echo "n1 rc=$?"; done
