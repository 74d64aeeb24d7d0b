CP_LIB=$PWD/exp/libconvpart_c1wtrace.so timeout 120 python scripts/c1w_trace.py > gpurun_out/r02v2_trace.txt 2>&1; echo "trace rc=$?"
