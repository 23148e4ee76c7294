# round 2: full GPU check of the build on a 2-GPU box: pytest -m gpu (multi-GPU included), smoke, bench N=1 and N=2
set -x
O=gpurun_out/r02full; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "EXIT $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "EXIT $?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_n1.jsonl 2> $O/bench_n1.err
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29601 bench.py --gpus 2 > $O/bench_n2.jsonl 2> $O/bench_n2.err
GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 29604 tools/step_trace.py > $O/trace_n2.txt 2>&1
