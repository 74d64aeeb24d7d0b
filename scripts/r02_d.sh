for v in default a b c; do
  if [ $v = default ]; then L=""; else L=$PWD/exp/libconvpart_fc$v.so; fi
  CP_LIB=$L timeout 300 python scripts/head_bench.py >> gpurun_out/r02d_head.jsonl 2>> gpurun_out/r02d_head.err; echo "$v rc=$?"
done
cat gpurun_out/r02d_head.jsonl
