# SGD of conv2 on the comm stream (overlapped with conv1 backward), conv1 SGD fused into its reduce
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02c_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c_pytest.log
timeout 300 python bench.py > gpurun_out/r02c_n1.json 2> gpurun_out/r02c_n1.err; echo "n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02c_n4.json 2> gpurun_out/r02c_n4.err; echo "n4 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02c_n2.json 2> gpurun_out/r02c_n2.err; echo "n2 rc=$?"
