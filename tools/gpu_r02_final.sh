# round 2 final check on a 2-GPU box: the driver's one-GPU view (pytest -m gpu, smoke, default bench),
# then N=2 momentum and BMUF lines of the final build
set -x
O=gpurun_out/r02final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu_1gpu.log 2>&1; echo "EXIT $?" >> $O/pytest_gpu_1gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "EXIT $?" >> $O/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $O/bench_n1.jsonl 2> $O/bench_n1.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.jsonl 2> $O/bench_ref.err
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 python bench.py --accum momentum --no-e2e --no-cpu-baseline > $O/bench_n1_mom.jsonl 2> $O/e1
timeout 600 $TR --master-port 29601 bench.py --gpus 2 --accum momentum --no-e2e --no-cpu-baseline > $O/bench_n2_mom.jsonl 2> $O/e2
timeout 600 $TR --master-port 29602 bench.py --gpus 2 --algo bmuf --no-e2e --no-cpu-baseline > $O/bench_n2_bmuf.jsonl 2> $O/e3
timeout 600 python bench.py --algo bmuf --no-e2e --no-cpu-baseline > $O/bench_n1_bmuf.jsonl 2> $O/e4
