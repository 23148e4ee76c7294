# round 2: prefetch stage of the ticketed step; bench hiccup (nvml / nvidia-smi)
set -x
O=gpurun_out/r02f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="bench.py --gpus 2 --warmup 20 --no-e2e --no-cpu-baseline"
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -x > $O/pytest_loopback.log 2>&1; echo "EXIT $?" >> $O/pytest_loopback.log
BENCH_NO_NVML=1 timeout 300 $TR --master-port 29601 $B --steps 200 > $O/bench_s200_nonvml.jsonl 2> $O/e1
BENCH_NO_SMI=1 timeout 300 $TR --master-port 29602 $B --steps 200 > $O/bench_s200_nosmi.jsonl 2> $O/e2
for cfg in "592 888" "592 1184" "296 592" "888 1184" "0 592"; do set -- $cfg
GTC_PREFETCH_LAG=$1 GTC_FUSED_LAG=$2 GTC_DECODE_TRACE=1 timeout 300 $TR --master-port 2960$(( $1 % 7 )) tools/step_trace.py > $O/trace_pf$1_la$2.txt 2>&1
done
