# pull reduce-scatter: parity (loopback pull/push, 2-4 GPU checks), then N=4/N=2 A/B push vs pull + graph phases
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02w_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tests/multi_gpu_check.py > gpurun_out/r02w_multi4.log 2>&1; echo "multi4 rc=$?"
for m in pull push; do CP_RS_MODE=$m timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02w_n4_$m.json 2> gpurun_out/r02w_n4_$m.err; echo "n4 $m rc=$?"; done
for m in pull push; do CP_RS_MODE=$m timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02w_n2_$m.json 2> gpurun_out/r02w_n2_$m.err; echo "n2 $m rc=$?"; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 scripts/graph_phases.py > gpurun_out/r02w_gphase_n4.jsonl 2> gpurun_out/r02w_gphase_n4.err; echo "gphase rc=$?"
