# A/B on one box: the ticketed kernel now (per-thread decode waits) vs the committed one (tools/exp_base)
set -x
O=gpurun_out/r02ab; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/base.so --csrc tools/exp_base >> $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for i in 1 2; do
GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 2960$i tools/step_trace.py > $O/trace_new$i.txt 2>&1
GTC_LIB=/tmp/base.so GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 2961$i tools/step_trace.py > $O/trace_base$i.txt 2>&1
done
