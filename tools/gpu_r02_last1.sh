# the driver's one-GPU view of the final tree: build, pytest -m gpu, smoke, default bench
set -x
O=${O:-gpurun_out/r02last2}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "EXIT $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "EXIT $?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_n1.jsonl 2> $O/bench_n1.err
timeout 300 python tools/sanitize_smoke.py > $O/sanitize_smoke.log 2>&1; echo "EXIT $?" >> $O/sanitize_smoke.log
