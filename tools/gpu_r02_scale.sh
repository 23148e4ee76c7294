# round 2: N = 1, 2, 4 lines of the final build on one 4-GPU box: fused (default),
# split and owner-computes at rho = 1 % and 10 %; torchrun parity at world 4
set -x
O=gpurun_out/r02scale; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench_n1.jsonl 2> $O/e_n1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --rho 0.1 > $O/bench_n1_rho10.jsonl 2> $O/e_n1r
p=29700
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
  for rho in 0.01 0.1; do
    for mode in fused split sharded; do
      extra=""; [ $mode = split ] && extra="--split-step"; [ $mode = sharded ] && extra="--sharded"
      p=$((p+1)); timeout 600 $TR --master-port $p bench.py --gpus $N --no-e2e --rho $rho $extra > $O/bench_n${N}_rho${rho}_$mode.jsonl 2> $O/e_n${N}_${rho}_$mode
    done
  done
  p=$((p+1)); timeout 600 $TR --master-port $p bench.py --gpus $N > $O/bench_n${N}.jsonl 2> $O/e_n${N}
  p=$((p+1)); GTC_DECODE_TRACE=1 timeout 300 $TR --master-port $p tools/step_trace.py > $O/trace_n${N}.txt 2>&1
done
timeout 1500 python -m pytest tests/test_multigpu.py -q > $O/pytest_multigpu_4gpu.log 2>&1; echo "EXIT $?" >> $O/pytest_multigpu_4gpu.log
