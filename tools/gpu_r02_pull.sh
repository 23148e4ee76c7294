# round 2: ticketed step with NVLink pulls instead of pushes (GTC_STEP_PULL=1)
set -x
O=gpurun_out/r02h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
GTC_STEP_PULL=1 GTC_PREFETCH_LAG=0 GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29604 tools/step_trace.py > $O/trace_pull.txt 2>&1
GTC_STEP_PULL=1 GTC_PREFETCH_LAG=0 GTC_FUSED_LAG=1184 GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29605 tools/step_trace.py > $O/trace_pull_la1184.txt 2>&1
GTC_STEP_PULL=1 GTC_PREFETCH_LAG=0 GTC_STEP_DIAG=2 GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29606 tools/step_trace.py > $O/trace_pull_noapply.txt 2>&1
