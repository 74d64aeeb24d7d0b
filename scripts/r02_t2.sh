# transposed forward chosen automatically for narrow slices: GPU suite, 4-rank check, bench N=1/2/4
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02t2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02t2_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tests/multi_gpu_check.py > gpurun_out/r02t2_multi4.log 2>&1; echo "multi4 rc=$?"; tail -1 gpurun_out/r02t2_multi4.log
timeout 300 python bench.py > gpurun_out/r02t2_n1.json 2> gpurun_out/r02t2_n1.err; echo "n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02t2_n2.json 2> gpurun_out/r02t2_n2.err; echo "n2 rc=$?"
for rep in 1 2; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02t2_n4_$rep.json 2> gpurun_out/r02t2_n4_$rep.err; echo "n4 rc=$?"; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29525 scripts/graph_phases.py > gpurun_out/r02t2_gphase_n4.jsonl 2> gpurun_out/r02t2_gphase_n4.err; echo "gphase4 rc=$?"
