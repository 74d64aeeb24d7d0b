# stream-tail finish variants chosen by pieces per unit: ncu at the slices, parity, N=4 / N=1 bench
for P in 1 4 8; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tail --csv \
    --log-file gpurun_out/r02t3_final_P$P.csv python scripts/pass_bench.py --P $P --reps 3 > gpurun_out/r02t3_final_P$P.log 2>&1; echo "P=$P rc=$?"
done
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02t3_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02t3_tests.log
for rep in 1 2; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02t3_n4_$rep.json 2> gpurun_out/r02t3_n4_$rep.err; echo "n4 rc=$?"; done
for rep in 1 2; do CP_LIB=exp/libconvpart_tailold.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 > gpurun_out/r02t3_n4old_$rep.json 2> gpurun_out/r02t3_n4old_$rep.err; echo "n4old rc=$?"; done
timeout 300 python bench.py > gpurun_out/r02t3_n1.json 2>/dev/null; echo "n1 rc=$?"
