# end-of-round validation on one box: GPU suite, smoke, bench N=1/2/4 (+ reference arm at N=1)
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; echo "n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/final_n2.json 2> gpurun_out/final_n2.err; echo "n2 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/final_n4.json 2> gpurun_out/final_n4.err; echo "n4 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"
