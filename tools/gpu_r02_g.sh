# round 2: bench without the NVML stall; finer phase trace of the ticketed step
set -x
O=gpurun_out/r02g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 2 --warmup 20 --no-e2e --no-cpu-baseline"
timeout 300 $TR --master-port 29601 $B --steps 1000 > $O/bench_n2.jsonl 2> $O/e1
GTC_PREFETCH_LAG=0 timeout 300 $TR --master-port 29602 $B --steps 1000 > $O/bench_n2_nopf.jsonl 2> $O/e2
GTC_STEP_KERNEL=grouped timeout 300 $TR --master-port 29603 $B --steps 1000 > $O/bench_n2_grouped.jsonl 2> $O/e3
GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29604 tools/step_trace.py > $O/trace.txt 2>&1
GTC_DECODE_TRACE=1 GTC_PREFETCH_LAG=0 timeout 300 $TR --master-port 29605 tools/step_trace.py > $O/trace_nopf.txt 2>&1
GTC_DECODE_TRACE=1 GTC_STEP_DIAG=2 timeout 300 $TR --master-port 29606 tools/step_trace.py > $O/trace_noapply.txt 2>&1
GTC_DECODE_TRACE=1 GTC_STEP_DIAG=4 timeout 300 $TR --master-port 29607 tools/step_trace.py > $O/trace_nodecode.txt 2>&1
