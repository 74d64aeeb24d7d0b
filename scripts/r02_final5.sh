# final round-2 validation on a 4-GPU box (HEAD after the reduce tweaks)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02K_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02K_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tests/multi_gpu_check.py > gpurun_out/r02K_multi4.log 2>&1; echo "multi4 rc=$?"; tail -1 gpurun_out/r02K_multi4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02K_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02K_smoke.log
for rep in 1 2; do timeout 300 python bench.py > gpurun_out/r02K_n1_$rep.json 2> gpurun_out/r02K_n1_$rep.err; echo "n1 rc=$?"; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r02K_n2.json 2> gpurun_out/r02K_n2.err; echo "n2 rc=$?"
for rep in 1 2; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02K_n4_$rep.json 2> gpurun_out/r02K_n4_$rep.err; echo "n4 rc=$?"; done
timeout 600 python bench.py --impl reference > gpurun_out/r02K_ref.json 2> gpurun_out/r02K_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02K_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r02K_ncu.log 2>&1; echo "ncu rc=$?"
