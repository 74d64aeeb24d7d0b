timeout 120 python scripts/conv1_bench.py > gpurun_out/r02v_conv1.jsonl 2>&1; echo "c1 rc=$?"
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r02v_all.log 2>&1; echo "all rc=$?"
timeout 300 python bench.py > gpurun_out/r02v_n1.json 2> gpurun_out/r02v_n1.err; echo "n1 rc=$?"
