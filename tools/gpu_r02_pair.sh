# experiment: the encode+push / decode kernel pair chained by PDL (GTC_STEP_PAIR=1) vs the ticketed kernel, N=2 and N=4
set -x
O=gpurun_out/r02pair; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
GTC_STEP_PAIR=1 timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "fused_step_parity" > $O/pytest_pair.log 2>&1; echo "EXIT $?" >> $O/pytest_pair.log
B="bench.py --gpus 2 --no-e2e --no-cpu-baseline --steps 1000"
p=29600
for rho in 0.01 0.1; do for i in 1 2; do
p=$((p+1)); GTC_STEP_PAIR=1 timeout 300 $TR2 --master-port $p $B --rho $rho > $O/bench_pair_${rho}_$i.jsonl 2> /dev/null
p=$((p+1)); timeout 300 $TR2 --master-port $p $B --rho $rho > $O/bench_tick_${rho}_$i.jsonl 2> /dev/null
done; done
