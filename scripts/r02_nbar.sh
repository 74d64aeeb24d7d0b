# conv1 forward: one polling warp + named barriers (nb) vs every warp polling (spin)
for v in spin nb spin nb; do
  CP_LIB=exp/libconvpart_$v.so timeout 120 python scripts/conv1_bench.py > gpurun_out/r02n_c1_$v.jsonl 2>&1; echo "$v rc=$?"
  python -c "
import json
for l in open('gpurun_out/r02n_c1_$v.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('$v', d['P'], round(d['new_ms']['fwd']*1e3,1), d['y_rel'], d['codes_diff'])
"
done
for v in spin nb; do for P in 1 4; do CP_LIB=exp/libconvpart_$v.so P=$P timeout 300 python scripts/slice_step.py > gpurun_out/r02n_${v}_P$P.json 2>&1; tail -1 gpurun_out/r02n_${v}_P$P.json; done; done
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_trajectory.py tests/test_gpu_full_size.py tests/test_gpu_loopback.py -x -q -m gpu > gpurun_out/r02n_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02n_tests.log
