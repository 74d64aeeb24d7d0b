# driver-like 1-GPU validation: GPU suite, smoke, bench N=1, reference arm
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02e_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02e_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02e_smoke.log
timeout 300 python bench.py > gpurun_out/r02e_n1.json 2> gpurun_out/r02e_n1.err; echo "n1 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02e_ref.json 2> gpurun_out/r02e_ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/r02e_ref.json
