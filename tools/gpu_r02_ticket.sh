# round 2: the ticketed fused step at N=2 -- parity (loopback + torchrun), bench vs the grouped kernel, lag sweep, trace
set -x
O=gpurun_out/r02t; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -x > $O/pytest_loopback.log 2>&1; echo "EXIT $?" >> $O/pytest_loopback.log
timeout 300 $TR --master-port 29601 bench.py --gpus 2 --steps 1000 --warmup 20 --no-e2e > $O/bench_n2.jsonl 2> $O/bench_n2.err
GTC_STEP_KERNEL=grouped timeout 300 $TR --master-port 29602 bench.py --gpus 2 --steps 1000 --warmup 20 --no-e2e > $O/bench_n2_grouped.jsonl 2> $O/bench_n2_grouped.err
for L in 148 296 1184 2368; do
GTC_FUSED_LAG=$L timeout 300 $TR --master-port 2961$((L % 7)) bench.py --gpus 2 --steps 1000 --warmup 20 --no-e2e > $O/bench_n2_lag$L.jsonl 2> $O/bench_n2_lag$L.err
done
GTC_DECODE_TRACE=1 TRACE_TAIL=8 timeout 300 $TR --master-port 29607 tools/step_trace.py > $O/trace_n2.txt 2>&1
GTC_STEP_KERNEL=grouped GTC_DECODE_TRACE=1 TRACE_TAIL=8 timeout 300 $TR --master-port 29608 tools/step_trace.py > $O/trace_n2_grouped.txt 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_multigpu.log 2>&1; echo "EXIT $?" >> $O/pytest_multigpu.log
