# conv1 wgrad with a separate raw-input ring (prefetch depth 4-5 chunks): timing + old-path comparison, parity
timeout 300 python scripts/conv1_bench.py > gpurun_out/r02o_c1.jsonl 2>&1; echo "c1 rc=$?"; grep "^{" gpurun_out/r02o_c1.jsonl
CP_C1W_RSTAGES=2 timeout 300 python scripts/conv1_bench.py > gpurun_out/r02o_c1_r2.jsonl 2>&1; echo "c1 r2 rc=$?"; grep "^{" gpurun_out/r02o_c1_r2.jsonl
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02o_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02o_pytest.log
