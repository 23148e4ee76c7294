# round 2: ticketed kernel at 4 / 5 / 6 CTAs per SM (registers 64 / 48 / 40), N=2
set -x
O=gpurun_out/r02t5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/lib_t5.so GTC_TICKET_CTAS=5 >> $O/build.log 2>&1 &
python tools/build_variant.py /tmp/lib_t6.so GTC_TICKET_CTAS=6 >> $O/build.log 2>&1 &
wait
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
export GTC_STEP_KERNEL=ticket
GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29604 tools/step_trace.py > $O/trace_t4.txt 2>&1
GTC_LIB=/tmp/lib_t5.so GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29605 tools/step_trace.py > $O/trace_t5.txt 2>&1
GTC_LIB=/tmp/lib_t6.so GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29606 tools/step_trace.py > $O/trace_t6.txt 2>&1
GTC_LIB=/tmp/lib_t5.so GTC_STEP_DIAG=6 GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29607 tools/step_trace.py > $O/trace_t5_nodecode.txt 2>&1
GTC_LIB=/tmp/lib_t5.so timeout 300 $TR --master-port 29601 bench.py --gpus 2 --warmup 20 --no-e2e --no-cpu-baseline --steps 1000 > $O/bench_t5.jsonl 2> $O/e1
timeout 300 $TR --master-port 29602 bench.py --gpus 2 --warmup 20 --no-e2e --no-cpu-baseline --steps 1000 > $O/bench_t4.jsonl 2> $O/e2
