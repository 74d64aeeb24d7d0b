# locate the CE-gather failure in the 4-rank check (progress on stderr), then N=2 A/B of the CE variants
CP_GATHER_MODE=ce timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tests/multi_gpu_check.py > gpurun_out/r02y_multi4_gce.log 2>&1; echo "multi4 gather-ce rc=$?"
grep "multi_gpu_check\]" gpurun_out/r02y_multi4_gce.log | tail -3
for m in "push push" "ce ce"; do set -- $m
  CP_RS_MODE=$1 CP_GATHER_MODE=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02y_n2_rs$1_g$2.json 2> gpurun_out/r02y_n2_rs$1_g$2.err; echo "n2 rs=$1 g=$2 rc=$?"; done
