# A/B on one box: the working tree vs the committed sources (tools/exp_base; build_variant --csrc), N=1 and N=2
set -x
O=gpurun_out/r02ab6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/build_variant.py /tmp/base.so --csrc tools/exp_base >> $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_parity.py tests/test_gpu_momentum.py -q -x > $O/pytest.log 2>&1; echo "EXIT $?" >> $O/pytest.log
B1="bench.py --no-e2e --no-cpu-baseline --steps 2000"
for i in 1 2; do
CUDA_VISIBLE_DEVICES=0 timeout 300 python $B1 > $O/bench1_new_$i.jsonl 2> /dev/null
CUDA_VISIBLE_DEVICES=0 GTC_LIB=/tmp/base.so timeout 300 python $B1 > $O/bench1_base_$i.jsonl 2> /dev/null
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 2 --no-e2e --no-cpu-baseline --steps 1000"
p=29600
for rho in 0.01 0.1; do for i in 1 2; do
p=$((p+1)); timeout 300 $TR --master-port $p $B --rho $rho > $O/bench_new_${rho}_$i.jsonl 2> /dev/null
p=$((p+1)); GTC_LIB=/tmp/base.so timeout 300 $TR --master-port $p $B --rho $rho > $O/bench_base_${rho}_$i.jsonl 2> /dev/null
done; done
