# multicast-cluster transposed forward (CP_TC_FWD_T=1 CP_TC_FWD_MC=1): timing at the slice shapes first (hang guard),
# then parity, then the 4-rank check and bench
set -x
for P in 4 8 2; do
  CP_TC_FWD_T=1 CP_TC_FWD_MC=1 timeout 90 python scripts/pass_bench.py --P $P --reps 10 >> gpurun_out/r02l_mc.jsonl 2>> gpurun_out/r02l_mc.err; echo "mc P=$P rc=$?"
  CP_TC_FWD_T=1 timeout 90 python scripts/pass_bench.py --P $P --reps 10 >> gpurun_out/r02l_t.jsonl 2>> gpurun_out/r02l_t.err; echo "fwdT P=$P rc=$?"
  timeout 90 python scripts/pass_bench.py --P $P --reps 10 >> gpurun_out/r02l_base.jsonl 2>> gpurun_out/r02l_base.err; echo "base P=$P rc=$?"
done
CP_TC_FWD_T=1 CP_TC_FWD_MC=1 timeout 600 python -m pytest tests/test_gpu_layers.py -x -q -k "forward_parity or split_forward or full_step" > gpurun_out/r02l_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02l_pytest.log
