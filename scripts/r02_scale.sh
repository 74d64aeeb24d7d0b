# N=1/2/4 bench lines on one 4-GPU box + N=1 launch list of the profiled step
timeout 300 python bench.py > gpurun_out/r02w_n1.json 2> gpurun_out/r02w_n1.err; echo "n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02w_n2.json 2> gpurun_out/r02w_n2.err; echo "n2 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02w_n4.json 2> gpurun_out/r02w_n4.err; echo "n4 rc=$?"
timeout 200 python scripts/prof_step.py > gpurun_out/r02w_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "step/" --csv --log-file gpurun_out/r02w_launches.csv python scripts/prof_step.py > gpurun_out/r02w_ncu.log 2>&1; echo "ncu rc=$?"
