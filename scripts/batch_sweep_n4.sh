# BASELINE configs[3] shape at the largest box available (4 GPUs): batch sweep with the Eq. 1
# (probe) partition, one bench line per batch
for b in 32 64 128 256 512 1024; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2956$((b % 10)) bench.py --gpus 4 --batch $b --partition probe --no-cpu-baseline 2>/dev/null | tail -1
done
