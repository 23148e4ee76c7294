# decode lag L (GTC_FUSED_LAG, default one wave = 740 at 5 CTAs/SM) and PDL on/off for the ticketed kernel:
# N=2 and N=4, rho 1 % and 10 %
set -x
O=gpurun_out/r02lag; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
p=29900
for N in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
B="bench.py --gpus $N --no-e2e --no-cpu-baseline --steps 1000"
for rho in 0.01 0.1; do
  for L in 370 555 740 1110 1480 2220; do
    p=$((p+1)); GTC_FUSED_LAG=$L timeout 300 $TR --master-port $p $B --rho $rho > $O/bench_n${N}_r${rho}_L$L.jsonl 2> /dev/null
  done
  p=$((p+1)); GTC_PDL=0 timeout 300 $TR --master-port $p $B --rho $rho > $O/bench_n${N}_r${rho}_nopdl.jsonl 2> /dev/null
done
done
