# transposed forward inside the fused 4-GPU step (P=4 slice: 0.187 vs 0.193 ms in LOCAL mode)
for v in 0 1 0 1; do CP_TC_FWD_T=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 >> gpurun_out/r02s2_n4.jsonl 2>> gpurun_out/r02s2_n4.err; echo "n4 fwdT=$v rc=$?"; done
