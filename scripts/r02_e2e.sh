# e2e with the network reading the staging buffers directly (no graph memcpy nodes)
for rep in 1 2; do timeout 300 python bench.py > gpurun_out/r02e_n1_$rep.json 2> gpurun_out/r02e_n1_$rep.err; echo "n1 rc=$?"; done
for rep in 1 2; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02e_n4_$rep.json 2> gpurun_out/r02e_n4_$rep.err; echo "n4 rc=$?"; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02e_n2.json 2> gpurun_out/r02e_n2.err; echo "n2 rc=$?"
