# RS variants push vs ce, gather kernel push vs copy engines, AR latency after the parallel-flag change
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02x_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29526 scripts/ar_bench.py > gpurun_out/r02x_ar4.txt 2>&1; echo "ar4 rc=$?"
CP_GATHER_MODE=ce timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tests/multi_gpu_check.py > gpurun_out/r02x_multi4_gce.log 2>&1; echo "multi4 gather-ce rc=$?"
for m in "push push" "ce push" "push ce" "ce ce"; do set -- $m
  CP_RS_MODE=$1 CP_GATHER_MODE=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02x_n4_rs$1_g$2.json 2> gpurun_out/r02x_n4_rs$1_g$2.err; echo "n4 rs=$1 g=$2 rc=$?"; done
