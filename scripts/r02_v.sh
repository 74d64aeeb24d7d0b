# N=4 overhead diagnostics: logits AllReduce latency, dgrad with local-only RS destinations, graph phases (split off)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29526 scripts/ar_bench.py > gpurun_out/r02v_ar4.txt 2>&1; echo "ar4 rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29527 scripts/ar_bench.py > gpurun_out/r02v_ar2.txt 2>&1; echo "ar2 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 scripts/graph_phases.py > gpurun_out/r02v_gphase_n4.jsonl 2> gpurun_out/r02v_gphase_n4.err; echo "gphase rc=$?"
CP_RS_LOCAL_DIAG=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29525 scripts/graph_phases.py > gpurun_out/r02v_gphase_n4_rslocal.jsonl 2> gpurun_out/r02v_gphase_n4_rslocal.err; echo "gphase rslocal rc=$?"
