# round 2, 2 GPUs: multi-process parity (incl. sharded), N=2 bench lines, fused-step phase trace
set -x
O=gpurun_out/r02n2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_multigpu.log 2>&1; echo "EXIT $?" >> $O/pytest_multigpu.log
timeout 300 $TR --master-port 29601 bench.py --gpus 2 --steps 1000 --warmup 20 > $O/bench_n2.jsonl 2> $O/bench_n2.err
timeout 300 $TR --master-port 29602 bench.py --gpus 2 --steps 1000 --warmup 20 --no-e2e --split-step > $O/bench_n2_split.jsonl 2> $O/bench_n2_split.err
timeout 300 $TR --master-port 29603 bench.py --gpus 2 --steps 1000 --warmup 20 --no-e2e --sharded > $O/bench_n2_sharded.jsonl 2> $O/bench_n2_sharded.err
timeout 300 $TR --master-port 29604 bench.py --gpus 2 --steps 500 --warmup 20 --no-e2e --rho 0.1 > $O/bench_n2_rho10.jsonl 2> $O/bench_n2_rho10.err
timeout 300 $TR --master-port 29605 bench.py --gpus 2 --steps 500 --warmup 20 --no-e2e --rho 0.1 --split-step > $O/bench_n2_rho10_split.jsonl 2> $O/bench_n2_rho10_split.err
timeout 300 $TR --master-port 29606 bench.py --gpus 2 --steps 500 --warmup 20 --no-e2e --rho 0.1 --sharded > $O/bench_n2_rho10_sharded.jsonl 2> $O/bench_n2_rho10_sharded.err
GTC_DECODE_TRACE=1 TRACE_TAIL=8 timeout 300 $TR --master-port 29607 tools/step_trace.py > $O/trace_n2.txt 2>&1
