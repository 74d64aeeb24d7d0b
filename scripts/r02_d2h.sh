# e2e: loss read-back as the e2e graph's last node (CP_BENCH_D2H_IN_GRAPH=1) vs a copy after the graph
for rep in 1 2; do for v in 0 1; do
  CP_BENCH_D2H_IN_GRAPH=$v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02d2_n1_${v}_$rep.json 2> gpurun_out/r02d2_n1_${v}_$rep.err; echo "n1 v=$v rc=$?"
  CP_BENCH_D2H_IN_GRAPH=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02d2_n4_${v}_$rep.json 2> gpurun_out/r02d2_n4_${v}_$rep.err; echo "n4 v=$v rc=$?"
done; done
