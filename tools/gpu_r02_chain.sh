# chained fused steps (default) vs GTC_STEP_CHAIN=0 on one box: torchrun parity (world 2), N=2 bench A/B at 1 % and 10 %, trace
set -x
O=gpurun_out/r02chain; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_multigpu.log 2>&1; echo "EXIT $?" >> $O/pytest_multigpu.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 2 --no-e2e --no-cpu-baseline --steps 1000"
p=29600
for rho in 0.01 0.1; do for i in 1 2; do
p=$((p+1)); timeout 300 $TR --master-port $p $B --rho $rho > $O/bench_chain_${rho}_$i.jsonl 2> $O/e_$p
p=$((p+1)); GTC_STEP_CHAIN=0 timeout 300 $TR --master-port $p $B --rho $rho > $O/bench_nochain_${rho}_$i.jsonl 2> $O/e_$p
done; done
p=$((p+1)); GTC_DECODE_TRACE=1 timeout 300 $TR --master-port $p tools/step_trace.py > $O/trace_chain.txt 2>&1
p=$((p+1)); timeout 300 $TR --master-port $p $B --accum momentum > $O/bench_chain_mom.jsonl 2> $O/e_mom
