# round 2 experiment: the two-stream step (GTC_STEP_2S=1) at N=2 -- parity (torchrun), trace-free timing, A/B with the default
set -x
O=gpurun_out/r02_2s; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
GTC_STEP_2S=1 timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "fused_step_parity" > $O/pytest_2s.log 2>&1; echo "EXIT $?" >> $O/pytest_2s.log
for i in 1 2; do
GTC_STEP_2S=1 timeout 300 $TR --master-port 2960$i bench.py --gpus 2 --no-e2e --no-cpu-baseline --steps 1000 > $O/bench_2s_$i.jsonl 2> $O/e2s$i
timeout 300 $TR --master-port 2961$i bench.py --gpus 2 --no-e2e --no-cpu-baseline --steps 1000 > $O/bench_def_$i.jsonl 2> $O/edef$i
done
