# split forward (256-multiple pair launch + transposed remainder) + deferred gather barrier: parity, pass times, N=4
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02u_pytest.log 2>&1; echo "pytest rc=$?"
for v in 0 1; do CP_TC_FWD_SPLIT=$v timeout 300 python scripts/pass_bench.py --P 4 --reps 10 >> gpurun_out/r02u_p4.jsonl 2>> gpurun_out/r02u_p4.err; echo "p4 split=$v rc=$?"; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tests/multi_gpu_check.py > gpurun_out/r02u_multi4.log 2>&1; echo "multi4 rc=$?"
for v in 1 0; do CP_TC_FWD_SPLIT=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02u_n4_s$v.json 2> gpurun_out/r02u_n4_s$v.err; echo "n4 split=$v rc=$?"; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29524 scripts/graph_phases.py > gpurun_out/r02u_gphase_n4.jsonl 2> gpurun_out/r02u_gphase_n4.err; echo "gphase rc=$?"
