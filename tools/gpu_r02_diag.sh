# round 2: ticketed step diagnostics at N=2 (ticket cost, apply cost, decode cost; bench vs trace timing gap)
set -x
O=gpurun_out/r02d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 2 --warmup 20 --no-e2e --no-cpu-baseline"
timeout 300 $TR --master-port 29601 $B --steps 200 > $O/bench_s200.jsonl 2> $O/e1
timeout 300 $TR --master-port 29602 $B --steps 1000 > $O/bench_s1000.jsonl 2> $O/e2
for D in 1 2 4 6 7; do
GTC_STEP_DIAG=$D timeout 300 $TR --master-port 2961$D $B --steps 1000 > $O/bench_diag$D.jsonl 2> $O/ed$D
done
GTC_STEP_KERNEL=grouped timeout 300 $TR --master-port 29620 $B --steps 1000 > $O/bench_grouped.jsonl 2> $O/e3
GTC_DECODE_TRACE=1 TRACE_STEPS=1000 timeout 300 $TR --master-port 29607 tools/step_trace.py > $O/trace_s1000.txt 2>&1
GTC_DECODE_TRACE=1 GTC_STEP_DIAG=1 timeout 300 $TR --master-port 29608 tools/step_trace.py > $O/trace_diag1.txt 2>&1
GTC_DECODE_TRACE=1 GTC_STEP_DIAG=6 timeout 300 $TR --master-port 29609 tools/step_trace.py > $O/trace_diag6.txt 2>&1
timeout 300 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu-baseline > $O/bench_n1.jsonl 2> $O/e4
