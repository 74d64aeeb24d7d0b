# f3 studies: the paper's four architectures at 1/2/4 GPUs, batch sweep at 1 GPU,
# Eq. 1 partitions from the probe and from injected (heterogeneous) device times.  One JSON line each.
cd $GRAFT_REPO_ROOT
out=gpurun_out/sweeps; mkdir -p $out
run1() { CUDA_VISIBLE_DEVICES=0 timeout 240 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1; }
runN() { n=$1; shift; timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+RANDOM%300)) bench.py --gpus $n --steps 10 --warmup 3 "$@" 2>/dev/null | tail -1; }
for net in 50:500 150:800 300:1000 500:1500; do
  run1 --net $net > $out/net_${net/:/-}_n1.json
  runN 2 --net $net > $out/net_${net/:/-}_n2.json
  runN 4 --net $net > $out/net_${net/:/-}_n4.json
done
for b in 32 64 256 512 1024; do run1 --batch $b > $out/batch_b${b}_n1.json; done
runN 4 --partition probe > $out/probe_n4.json
runN 4 --batch 512 > $out/batch_b512_n4.json
runN 4 --probe-times 1,1,1.5,2 > $out/injected_1-1-1.5-2_n4.json
runN 2 --probe-times 1,2 > $out/injected_1-2_n2.json
run1 --lrn > $out/lrn_n1.json
runN 4 --lrn > $out/lrn_n4.json
