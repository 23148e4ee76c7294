# round 2 experiment: gpu-scope first loads / entry stores in the ticketed kernel (N=2 trace)
set -x
O=gpurun_out/r02scope; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/lib_scope.so GTC_SCOPE_EXP >> $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29604 tools/step_trace.py > $O/trace_sys.txt 2>&1
GTC_LIB=/tmp/lib_scope.so GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29605 tools/step_trace.py > $O/trace_gpu.txt 2>&1
GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29606 tools/step_trace.py > $O/trace_sys2.txt 2>&1
GTC_LIB=/tmp/lib_scope.so GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29607 tools/step_trace.py > $O/trace_gpu2.txt 2>&1
