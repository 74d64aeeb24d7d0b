# conv1 forward (set, M tile) unit balancing A/B (CP_C1_BALANCE), parity, step-level effect
mkdir -p gpurun_out
for b in 0 1 0 1; do CP_C1_BALANCE=$b timeout 120 python scripts/conv1_bench.py > gpurun_out/r02bal_conv1_b$b.jsonl 2>&1; echo "c1 b=$b rc=$?"; cat gpurun_out/r02bal_conv1_b$b.jsonl | head -2; done
timeout 600 python -m pytest tests/test_gpu_layers.py -x -q -m gpu -k "unit_split or forward_parity or fused_sgd" > gpurun_out/r02bal_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02bal_tests.log
timeout 600 python -m pytest tests/test_gpu_full_size.py tests/test_gpu_trajectory.py -x -q -m gpu > gpurun_out/r02bal_full.log 2>&1; echo "full rc=$?"; tail -2 gpurun_out/r02bal_full.log
for b in 0 1 0 1; do CP_C1_BALANCE=$b timeout 300 python bench.py > gpurun_out/r02bal_n1_b$b.json 2>/dev/null; echo "n1 b=$b rc=$?"; python -c "import json;d=json.load(open('gpurun_out/r02bal_n1_b$b.json'));print(d['value'],d['ms_per_step'],d['clocks']['sm_mhz'])"; done
