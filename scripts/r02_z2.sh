CP_LIB=$PWD/exp/libconvpart_c1ftrace2.so timeout 120 python scripts/c1f_trace.py > gpurun_out/r02z2_c1ftrace.txt 2>&1; echo "trace rc=$?"; grep c1f_trace gpurun_out/r02z2_c1ftrace.txt | tail -12
timeout 300 python scripts/conv1_bench.py > gpurun_out/r02z2_c1.jsonl 2>&1; echo "c1 rc=$?"; grep "^{" gpurun_out/r02z2_c1.jsonl | cut -c1-200
CP_C1_PAD=0 timeout 300 python scripts/conv1_bench.py > gpurun_out/r02z2_c1_nopad.jsonl 2>&1; echo "c1 nopad rc=$?"; grep "^{" gpurun_out/r02z2_c1_nopad.jsonl | cut -c1-200
