# conv2 pass times at the P=1/2/4/8 slice shapes (rank 0's slice, LOCAL mode, 1 GPU), N=4 phase times,
# NVML NVLink counter probe, multicast + 2 push warps at N=4
for P in 1 2 4 8; do timeout 300 python scripts/pass_bench.py --P $P --reps 10 >> gpurun_out/r02s_slices.jsonl 2>> gpurun_out/r02s_slices.err; echo "P=$P rc=$?"; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 scripts/phase_times.py > gpurun_out/r02s_phase_n4.jsonl 2> gpurun_out/r02s_phase_n4.err; echo "phase rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29525 scripts/nvml_nvlink_probe.py > gpurun_out/r02s_nvml2.txt 2>&1; echo "nvml rc=$?"
CP_MULTICAST=1 CP_TC_PUSH_WARPS=2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02s_n4_mc1pw2.json 2> gpurun_out/r02s_n4_mc1pw2.err; echo "n4 mc pw2 rc=$?"
