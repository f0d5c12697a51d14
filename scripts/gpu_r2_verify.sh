# round-2 re-entry check: full GPU suite, smoke(), default bench line, host info
mkdir -p gpurun_out
echo "nproc $(nproc)"; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-600
