# transposed forward in the 4-GPU bench (fused collectives): auto (on at P=4) vs forced off
for t in 1 0 1; do
  CP_TC_FWD_T=$t timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2951$t bench.py --gpus 4 --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fwdT=$t', round(d['value']), d['ms_per_step'], d['roofline']['kernel_ms_live'], d['clocks']['sm_mhz'])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 tests/multi_gpu_check.py > gpurun_out/fwdT_multi.log 2>&1; echo "multi rc=$?"
