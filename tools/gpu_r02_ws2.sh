set -x
O=gpurun_out/r02w8; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_loopback.py -q -x -k "fused" > $O/pytest_loopback.log 2>&1; echo "EXIT $?" >> $O/pytest_loopback.log
GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29604 tools/step_trace.py > $O/trace.txt 2>&1
timeout 300 $TR --master-port 29601 bench.py --gpus 2 --warmup 20 --no-e2e --no-cpu-baseline --steps 1000 > $O/bench_n2.jsonl 2> $O/e1
