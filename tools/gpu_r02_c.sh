set -x
O=gpurun_out/r02c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -x > $O/pytest_loopback.log 2>&1; echo "EXIT $?" >> $O/pytest_loopback.log
GTC_C5_REPORT=$O/c5.json timeout 900 python -m pytest tests/test_gpu_c5.py -q -s > $O/c5.log 2>&1; echo "EXIT $?" >> $O/c5.log
timeout 300 python tools/gradnull_timing.py > $O/gradnull.log 2>&1
