# fused p2p step phase trace at N=2 (tail detail)
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29610 tools/step_trace.py"
GTC_DECODE_TRACE=1 TRACE_TAIL=30 timeout 300 $T > gpurun_out/trace_n2.txt 2>&1
