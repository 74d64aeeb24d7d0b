# rank-order sum of the copy-engine reduce-scatter on a small grid-stride grid (32 x 512) vs the former flood
for rep in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02j_n4_$rep.json 2> gpurun_out/r02j_n4_$rep.err; echo "n4 rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02j_n2.json 2> gpurun_out/r02j_n2.err; echo "n2 rc=$?"
CP_RS_SUM_BLOCKS=8 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02j_n2_b8.json 2> gpurun_out/r02j_n2_b8.err; echo "n2 b8 rc=$?"
CP_RS_SUM_BLOCKS=128 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02j_n2_b128.json 2> gpurun_out/r02j_n2_b128.err; echo "n2 b128 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29524 scripts/graph_phases.py > gpurun_out/r02j_gphase_n2.jsonl 2> gpurun_out/r02j_gphase_n2.err; echo "gphase2 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tests/multi_gpu_check.py > gpurun_out/r02j_multi4.log 2>&1; echo "multi4 rc=$?"; tail -1 gpurun_out/r02j_multi4.log
