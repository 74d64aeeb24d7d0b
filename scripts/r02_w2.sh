CP_LIB=$PWD/exp/libconvpart_c1wtrace_a8.so timeout 120 python scripts/c1w_trace.py > gpurun_out/r02w2_trace_a8.txt 2>&1; echo "trace a8 rc=$?"
CP_LIB=$PWD/exp/libconvpart_c1w_a8.so timeout 300 python scripts/conv1_bench.py > gpurun_out/r02w2_c1_a8.jsonl 2>&1; echo "c1 a8 rc=$?"; grep "^{" gpurun_out/r02w2_c1_a8.jsonl | cut -c1-200
timeout 300 python scripts/conv1_bench.py > gpurun_out/r02w2_c1_a4.jsonl 2>&1; echo "c1 a4 rc=$?"; grep "^{" gpurun_out/r02w2_c1_a4.jsonl | cut -c1-200
