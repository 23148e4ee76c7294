# round 2: full GPU check of the build on a 2-GPU box + N=1 / N=2 bench lines
set -x
O=gpurun_out/r02check2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "EXIT $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "EXIT $?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_n1.jsonl 2> $O/bench_n1.err
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29601 bench.py --gpus 2 > $O/bench_n2.jsonl 2> $O/bench_n2.err
timeout 600 $TR --master-port 29602 bench.py --gpus 2 --impl reference --steps 5 --warmup 3 > $O/bench_n2_ref.jsonl 2> $O/bench_n2_ref.err
