# what the driver runs at round end on one GPU: pytest -m gpu, smoke, bench
mkdir -p gpurun_out/final1
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/final1/pytest_gpu_1gpu.log 2>&1; echo "EXIT $?" >> gpurun_out/final1/pytest_gpu_1gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final1/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final1/bench_n1.jsonl 2> gpurun_out/final1/bench_n1.err
