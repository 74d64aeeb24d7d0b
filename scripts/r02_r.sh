for c in 1 0 3 4; do CP_FC_CPB=$c timeout 300 python scripts/head_bench.py 2>&1 | tail -1 | sed "s/^/cpb=$c /"; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02r_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02r_pytest.log
for rep in 1 2; do timeout 300 python bench.py > gpurun_out/r02r_n1_$rep.json 2> gpurun_out/r02r_n1_$rep.err; echo "n1 rc=$?"; done
