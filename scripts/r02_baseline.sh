# round-2 baseline on a 2-GPU box: GPU suite (incl. the 2-rank check), bench N=1 and N=2
nvidia-smi -L > gpurun_out/r02b_smi.txt
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r02b_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py > gpurun_out/r02b_n1.json 2> gpurun_out/r02b_n1.err; echo "n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02b_n2.json 2> gpurun_out/r02b_n2.err; echo "n2 rc=$?"
