# round 2: shapes of the warp-specialized kernel (CTAs/SM x encode groups x decode warps), N=2 trace
set -x
O=gpurun_out/r02w12; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/lib_3g8w.so GTC_WS_GROUPS=3 GTC_WS_DECW=8 GTC_WS_CTAS=1 >> $O/build.log 2>&1 &
wait
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29604 tools/step_trace.py > $O/trace_2x2g2w.txt 2>&1
for v in 3g8w; do
GTC_LIB=/tmp/lib_$v.so GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29605 tools/step_trace.py > $O/trace_1x$v.txt 2>&1
done
GTC_LIB=/tmp/lib_3g8w.so timeout 600 python -m pytest tests/test_gpu_loopback.py -q -x -k "fused" > $O/pytest_loopback_3g8w.log 2>&1; echo "EXIT $?" >> $O/pytest_loopback_3g8w.log
timeout 600 python -m pytest tests/test_gpu_loopback.py -q -x -k "fused" > $O/pytest_loopback.log 2>&1; echo "EXIT $?" >> $O/pytest_loopback.log
