# the ticketed kernel at 4 / 5 / 6 CTAs per SM after the diet: N=2 and N=4, 1 %; parity of the 5-CTA build
set -x
O=gpurun_out/r02t5c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/t5.so GTC_TICKET_CTAS=5 >> $O/build.log 2>&1 &
python tools/build_variant.py /tmp/t6.so GTC_TICKET_CTAS=6 >> $O/build.log 2>&1 &
wait
GTC_LIB=/tmp/t5.so timeout 900 python -m pytest tests/test_gpu_loopback.py -q -x > $O/pytest_loopback_t5.log 2>&1; echo "EXIT $?" >> $O/pytest_loopback_t5.log
p=29600
for N in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
B="bench.py --gpus $N --no-e2e --no-cpu-baseline --steps 1000"
for v in t4 t5 t6; do
  L=""; [ $v = t5 ] && L="/tmp/t5.so"; [ $v = t6 ] && L="/tmp/t6.so"
  p=$((p+1)); GTC_LIB=$L timeout 300 $TR --master-port $p $B > $O/bench_n${N}_$v.jsonl 2> /dev/null
done
p=$((p+1)); GTC_LIB=/tmp/t5.so timeout 300 $TR --master-port $p $B --accum momentum > $O/bench_n${N}_t5_mom.jsonl 2> /dev/null
p=$((p+1)); timeout 300 $TR --master-port $p $B --accum momentum > $O/bench_n${N}_t4_mom.jsonl 2> /dev/null
done
GTC_LIB=/tmp/t5.so timeout 1500 python -m pytest tests/test_multigpu.py -q -x -k "fused or momentum" > $O/pytest_multigpu_t5.log 2>&1; echo "EXIT $?" >> $O/pytest_multigpu_t5.log
