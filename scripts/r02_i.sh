# fused logits AllReduce + softmax: GPU suite (multi-GPU parity), 4-rank check, bench N=4/N=2, graph phases N=4
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02i_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02i_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tests/multi_gpu_check.py > gpurun_out/r02i_multi4.log 2>&1; echo "multi4 rc=$?"; tail -1 gpurun_out/r02i_multi4.log
for rep in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02i_n4_$rep.json 2> gpurun_out/r02i_n4_$rep.err; echo "n4 rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02i_n2.json 2> gpurun_out/r02i_n2.err; echo "n2 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29525 scripts/graph_phases.py > gpurun_out/r02i_gphase_n4.jsonl 2> gpurun_out/r02i_gphase_n4.err; echo "gphase4 rc=$?"
