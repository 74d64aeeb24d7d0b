timeout 300 python scripts/head_bench.py > gpurun_out/r02n_head.jsonl 2>&1; echo "head rc=$?"; cat gpurun_out/r02n_head.jsonl | tail -1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02n_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02n_pytest.log
for rep in 1 2; do timeout 300 python bench.py > gpurun_out/r02n_n1_$rep.json 2> gpurun_out/r02n_n1_$rep.err; echo "n1 rc=$?"; done
