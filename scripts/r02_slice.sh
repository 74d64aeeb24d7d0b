# per-kernel launch list of one rank's compute at P=4 / P=8 (compute-only step on one GPU)
for P in 4 8; do
  P=$P timeout 300 python scripts/slice_step.py > gpurun_out/r02s_P$P.json 2>&1; echo "P=$P rc=$?"; cat gpurun_out/r02s_P$P.json | tail -1
  P=$P STEPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02s_launches_P$P.csv python scripts/slice_step.py > gpurun_out/r02s_ncu_P$P.log 2>&1; echo "ncu P=$P rc=$?"
done
