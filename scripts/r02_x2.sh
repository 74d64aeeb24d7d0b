CP_LIB=$PWD/exp/libconvpart_c1w_a12.so timeout 300 python scripts/conv1_bench.py > gpurun_out/r02x2_c1_a12.jsonl 2>&1; echo "c1 a12 rc=$?"; grep "^{" gpurun_out/r02x2_c1_a12.jsonl | cut -c1-190
timeout 300 python scripts/conv1_bench.py > gpurun_out/r02x2_c1_a8.jsonl 2>&1; echo "c1 a8 (default) rc=$?"; grep "^{" gpurun_out/r02x2_c1_a8.jsonl | cut -c1-190
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02x2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02x2_pytest.log
