# final-state bench lines N=1/2/4 (e2e prefetch reorder), twice each for the spread
for rep in 1 2; do
timeout 300 python bench.py > gpurun_out/r02f_n1_$rep.json 2> gpurun_out/r02f_n1_$rep.err; echo "n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02f_n2_$rep.json 2> gpurun_out/r02f_n2_$rep.err; echo "n2 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02f_n4_$rep.json 2> gpurun_out/r02f_n4_$rep.err; echo "n4 rc=$?"
done
