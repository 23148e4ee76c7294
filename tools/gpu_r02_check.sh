# round 2: loopback parity first, then the rest of -m gpu, smoke and a short bench
set -x
mkdir -p gpurun_out/r02a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02a/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -x > gpurun_out/r02a/pytest_loopback.log 2>&1; echo "EXIT $?" >> gpurun_out/r02a/pytest_loopback.log
timeout 1200 python -m pytest tests -q -m gpu --deselect tests/test_gpu_loopback.py > gpurun_out/r02a/pytest_gpu.log 2>&1; echo "EXIT $?" >> gpurun_out/r02a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.log 2>&1
timeout 600 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/r02a/bench_n1.jsonl 2> gpurun_out/r02a/bench_n1.err
