# transposed forward: parity (layer variants incl. P=1/2/3, full size), then pass times on/off
CP_TC_FWD_T=1 timeout 600 python -m pytest tests/test_gpu_layers.py tests/test_gpu_full_size.py -x -q -k "forward or full_step or full_size or variants" > gpurun_out/fwdT_tests.log 2>&1
echo "tests rc=$?"
for P in 1 2 4 8; do
  for t in 1 0; do
    echo "fwdT=$t P=$P $(CP_TC_FWD_T=$t timeout 100 python scripts/pass_bench.py --P $P --reps 20 2>&1 | tail -1 | grep -o '"fwd": [0-9.]*' | head -1)"
  done
done
