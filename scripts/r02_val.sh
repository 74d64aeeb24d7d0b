# validation on 2 GPUs: GPU suite (incl. 2-rank check), bench N=1 and N=2
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r02o_all.log 2>&1; echo "all rc=$?"
timeout 300 python bench.py > gpurun_out/r02o_n1.json 2> gpurun_out/r02o_n1.err; echo "n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02o_n2.json 2> gpurun_out/r02o_n2.err; echo "n2 rc=$?"
