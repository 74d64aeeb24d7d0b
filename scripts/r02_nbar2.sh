# conv1 forward named-barrier A/B with ncu durations (CUDA events here tick in 2.048 us)
for v in spin nb spin nb; do for P in 1 4; do
  CP_LIB=exp/libconvpart_$v.so P=$P STEPS=4 timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:conv1_fwd --csv --log-file gpurun_out/r02n2_${v}_P${P}_$RANDOM.csv python scripts/slice_step.py > /dev/null 2>&1; echo "$v P=$P rc=$?"
done; done
