# fused p2p step phase trace at N=2: default lag; lag = T (encode wave, then decode wave); weak stores
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29610 tools/step_trace.py"
GTC_DECODE_TRACE=1 GTC_FUSED_LAG=5930 timeout 300 $T > gpurun_out/trace_n2_lagT.txt 2>&1
GTC_DECODE_TRACE=1 GTC_FUSED_LAG=5930 GTC_FUSED_WEAK=1 timeout 300 $T > gpurun_out/trace_n2_lagT_weak.txt 2>&1
GTC_DECODE_TRACE=1 GTC_FUSED_WEAK=1 timeout 300 $T > gpurun_out/trace_n2_weak.txt 2>&1
