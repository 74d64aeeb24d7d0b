CP_GATHER_MODE=ce timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29528 scripts/ce_repro.py > gpurun_out/r02z_ce_repro.log 2>&1; echo "repro rc=$?"
grep "^\[r" gpurun_out/r02z_ce_repro.log | head -40
