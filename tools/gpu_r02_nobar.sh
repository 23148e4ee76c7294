# round 2: ticketed kernel with per-thread decode waits (one barrier less); parity + N=2 trace/bench
set -x
O=gpurun_out/r02nobar; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -x > $O/pytest_loopback.log 2>&1; echo "EXIT $?" >> $O/pytest_loopback.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29604 tools/step_trace.py > $O/trace.txt 2>&1
timeout 600 $TR --master-port 29601 bench.py --gpus 2 --no-e2e --no-cpu-baseline > $O/bench_n2.jsonl 2> $O/e1
timeout 600 $TR --master-port 29602 bench.py --gpus 2 --no-e2e --no-cpu-baseline --rho 0.1 > $O/bench_n2_rho10.jsonl 2> $O/e2
timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "fused or momentum" > $O/pytest_multigpu.log 2>&1; echo "EXIT $?" >> $O/pytest_multigpu.log
