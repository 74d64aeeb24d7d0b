# round-2 parity additions on a 2-GPU box: new 1-GPU tests, then the whole GPU suite (incl. 2-rank check)
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_trajectory.py tests/test_gpu_layers.py -x -q -k "loopback or trajectory or image_dgrad" -s > gpurun_out/r02p_new.log 2>&1; echo "new rc=$?"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02p_all.log 2>&1; echo "all rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02p_n2.json 2> gpurun_out/r02p_n2.err; echo "n2 rc=$?"
