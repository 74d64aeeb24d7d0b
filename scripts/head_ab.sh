# partitioned vs replicated FC head at N=2/4 (fused collectives), alternating
for n in 4 2; do
for h in partitioned replicated partitioned replicated; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --head $h --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n=$n', '$h', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
