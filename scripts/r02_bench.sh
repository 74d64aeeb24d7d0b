# bench N=1, N=2, reference arm (new bench fields)
timeout 600 python bench.py > gpurun_out/r02c_n1.json 2> gpurun_out/r02c_n1.err; echo "n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02c_n2.json 2> gpurun_out/r02c_n2.err; echo "n2 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r02c_ref.json 2> gpurun_out/r02c_ref.err; echo "ref rc=$?"
