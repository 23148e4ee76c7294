# Round-end regression + measurement on 4 GPUs: the full GPU suite, smoke,
# bench lines at N=1/2/4 (fused p2p step and separate kernels), the 1e9
# config, and the N=1 ncu launch list + full capture of the step kernel.
set -x
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/final/pytest_gpu_4gpu.log 2>&1; echo "EXIT $?" >> gpurun_out/final/pytest_gpu_4gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final/bench_n1.jsonl 2> gpurun_out/final/bench_n1.err
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 400 $R --nproc-per-node $N --master-port 2960$N bench.py --gpus $N > gpurun_out/final/bench_n$N.jsonl 2> gpurun_out/final/bench_n$N.err
  GTC_STEP_FUSED=0 timeout 400 $R --nproc-per-node $N --master-port 2961$N bench.py --gpus $N --no-e2e > gpurun_out/final/bench_n${N}_unfused.jsonl 2>/dev/null
done
timeout 600 $R --nproc-per-node 4 --master-port 29620 bench.py --gpus 4 --workload 1e9 --steps 20 --warmup 3 --no-e2e > gpurun_out/final/bench_n4_1e9.jsonl 2> gpurun_out/final/bench_n4_1e9.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_n1.csv python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gtc_encode_tile_kernel -s 20 -c 1 -o gpurun_out/final/ncu_full_n1 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final/ncu_full.log 2>&1
ls -la gpurun_out/final
