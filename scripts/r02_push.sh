# gather push warps A/B at N=2 and N=4 (4-GPU box)
for v in 1 2; do CP_TC_PUSH_WARPS=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02y_n4_pw$v.json 2> gpurun_out/r02y_n4_pw$v.err; echo "n4 pw=$v rc=$?"; done
for v in 1 2; do CP_TC_PUSH_WARPS=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02y_n2_pw$v.json 2> gpurun_out/r02y_n2_pw$v.err; echo "n2 pw=$v rc=$?"; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tests/multi_gpu_check.py > gpurun_out/r02y_multi4.log 2>&1; echo "multi4 rc=$?"
python scripts/mc_probe.py > gpurun_out/r02y_mc.txt 2>&1; cat /proc/sys/kernel/yama/ptrace_scope >> gpurun_out/r02y_mc.txt 2>&1; nvidia-smi -q | grep -i -A3 "fabric" >> gpurun_out/r02y_mc.txt 2>&1; echo "mc rc=$?"
