# two copy streams for the copy-engine gather / reduce-scatter: parity at 4 ranks, then N=4 / N=2 A/B
CP_GATHER_CE_STREAMS=2 CP_RS_CE_STREAMS=2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 tests/multi_gpu_check.py > gpurun_out/r02p_multi4.log 2>&1; echo "multi4 rc=$?"; tail -1 gpurun_out/r02p_multi4.log
for v in "1 1" "2 1" "1 2" "2 2" "1 1" "2 2"; do set -- $v
  CP_GATHER_CE_STREAMS=$1 CP_RS_CE_STREAMS=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 >> gpurun_out/r02p_n4.jsonl 2> gpurun_out/r02p_n4.err; echo "n4 $1 $2 rc=$?"
done
for v in "1 1" "2 2"; do set -- $v
  CP_GATHER_CE_STREAMS=$1 CP_RS_CE_STREAMS=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 >> gpurun_out/r02p_n2.jsonl 2> gpurun_out/r02p_n2.err; echo "n2 $1 $2 rc=$?"
done
