# the scaled network (BASELINE configs[4]: 512:2048 on 224x224, batch 256) on the round-2 build
timeout 900 python bench.py --net scaled --batch 256 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02sc_n1.json 2> gpurun_out/r02sc_n1.err; echo "n1 rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 --net scaled --batch 256 --steps 5 --warmup 3 > gpurun_out/r02sc_n4.json 2> gpurun_out/r02sc_n4.err; echo "n4 rc=$?"
