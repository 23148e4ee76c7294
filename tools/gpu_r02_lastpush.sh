# A/B: the last wave's pushes waited to completion (GTC_LAST_PUSH_FULL) vs read-only waits, N=2 traces (launch gap)
set -x
O=gpurun_out/r02lp; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/lp.so GTC_LAST_PUSH_FULL >> $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for i in 1 2; do
GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 2960$i tools/step_trace.py > $O/trace_def$i.txt 2>&1
GTC_LIB=/tmp/lp.so GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 2961$i tools/step_trace.py > $O/trace_lp$i.txt 2>&1
done
