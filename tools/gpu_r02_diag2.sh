# round 2: bench warm-up right before timing; inter-kernel gap of the fused step (pushes, PDL)
set -x
O=gpurun_out/r02e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 2 --warmup 20 --no-e2e --no-cpu-baseline"
timeout 300 $TR --master-port 29601 $B --steps 200 > $O/bench_s200.jsonl 2> $O/e1
timeout 300 $TR --master-port 29602 $B --steps 1000 > $O/bench_s1000.jsonl 2> $O/e2
GTC_STEP_KERNEL=grouped timeout 300 $TR --master-port 29603 $B --steps 1000 > $O/bench_grouped.jsonl 2> $O/e3
GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29607 tools/step_trace.py > $O/trace.txt 2>&1
GTC_DECODE_TRACE=1 GTC_STEP_DIAG=16 timeout 300 $TR --master-port 29608 tools/step_trace.py > $O/trace_nopush.txt 2>&1
GTC_DECODE_TRACE=1 GTC_STEP_DIAG=22 timeout 300 $TR --master-port 29609 tools/step_trace.py > $O/trace_encode_only.txt 2>&1
GTC_DECODE_TRACE=1 GTC_PDL=0 timeout 300 $TR --master-port 29610 tools/step_trace.py > $O/trace_nopdl.txt 2>&1
timeout 300 python bench.py --steps 200 --warmup 20 --no-e2e --no-cpu-baseline > $O/bench_n1_s200.jsonl 2> $O/e4
