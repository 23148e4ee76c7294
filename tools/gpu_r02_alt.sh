# final tree: lag fine-tuning around 1.5 waves, and the split / owner-computes paths at N=2 and N=4
set -x
O=gpurun_out/r02alt; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
p=29950
for N in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
B="bench.py --gpus $N --no-e2e --no-cpu-baseline --steps 1000"
for rho in 0.01 0.1; do
  for L in 925 1110 1295; do
    p=$((p+1)); GTC_FUSED_LAG=$L timeout 300 $TR --master-port $p $B --rho $rho > $O/bench_n${N}_r${rho}_L$L.jsonl 2> /dev/null
  done
  p=$((p+1)); timeout 300 $TR --master-port $p $B --rho $rho --split-step > $O/bench_n${N}_r${rho}_split.jsonl 2> $O/e_split_$N_$rho
  p=$((p+1)); timeout 300 $TR --master-port $p $B --rho $rho --sharded > $O/bench_n${N}_r${rho}_sharded.jsonl 2> $O/e_sh_$N_$rho
done
done
