# NVLink multicast gather A/B (4-GPU box) + full GPU suite (covers the FC head kernels)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02mc_pytest.log 2>&1; echo "pytest rc=$?"
CP_MULTICAST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tests/multi_gpu_check.py > gpurun_out/r02mc_multi4.log 2>&1; echo "multi4 mc rc=$?"
for v in 0 1; do CP_MULTICAST=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02mc_n4_mc$v.json 2> gpurun_out/r02mc_n4_mc$v.err; echo "n4 mc=$v rc=$?"; done
for v in 0 1; do CP_MULTICAST=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02mc_n2_mc$v.json 2> gpurun_out/r02mc_n2_mc$v.err; echo "n2 mc=$v rc=$?"; done
timeout 300 python bench.py > gpurun_out/r02mc_n1.json 2> gpurun_out/r02mc_n1.err; echo "n1 rc=$?"
