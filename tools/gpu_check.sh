# Re-entry check: GPU tests, default bench, reference arm.
mkdir -p gpurun_out/chk
python -m pytest tests -m gpu -x -q > gpurun_out/chk/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/chk/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk/smoke.log 2>&1
python bench.py > gpurun_out/chk/bench.log 2> gpurun_out/chk/bench.err
tail -3 gpurun_out/chk/pytest.log; cat gpurun_out/chk/bench.log | head -c 3000
