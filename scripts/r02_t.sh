# conv1 forward limiter experiments (C1_EXP builds), bench N=1 and N=4 (pipelined e2e graph), ncu full step
for n in 0 1 2 3 4; do
  if [ $n = 0 ]; then L=""; else L=$PWD/exp/libconvpart_c1e$n.so; fi
  CP_LIB=$L timeout 300 python scripts/conv1_bench.py > gpurun_out/r02t_c1e$n.jsonl 2>&1; echo "c1e$n rc=$?"
done
timeout 300 python bench.py > gpurun_out/r02t_n1.json 2> gpurun_out/r02t_n1.err; echo "n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02t_n4.json 2> gpurun_out/r02t_n4.err; echo "n4 rc=$?"
timeout 300 python scripts/prof_step.py > gpurun_out/r02t_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" -o gpurun_out/r02t_step python scripts/prof_step.py > gpurun_out/r02t_ncu.log 2>&1; echo "ncu rc=$?"
