# fwd halo A boxes: parity (layers, full step, full size, planner variants), then pass times on/off
CP_NVCC_EXTRA=-DCP_TC_HALO_HOOK python -c "from paper_1712_02546_b200 import build; build.build(force=True)"
CP_TC_FWD_HALO=1 timeout 600 python -m pytest tests/test_gpu_layers.py tests/test_gpu_full_size.py -x -q > gpurun_out/halo_tests.log 2>&1
echo "tests rc=$?"
for P in 1 2 4; do
  for h in 1 0; do
    echo "halo=$h P=$P $(CP_TC_FWD_HALO=$h timeout 100 python scripts/pass_bench.py --P $P --reps 20 2>&1 | tail -1 | cut -c100-300)"
  done
done
