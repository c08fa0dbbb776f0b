# Round 2 first GPU check: tests, smoke, bench, regrid host profile.
mkdir -p gpurun_out/r2a
python -m pytest tests -m gpu -x -q > gpurun_out/r2a/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2a/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1
python bench.py > gpurun_out/r2a/bench.log 2> gpurun_out/r2a/bench.err
timeout 600 python tools/prof_regrid.py > gpurun_out/r2a/regrid.log 2>&1
tail -3 gpurun_out/r2a/pytest.log; head -c 1500 gpurun_out/r2a/bench.log
