# one GPU iteration: targeted tests (PYTESTSEL), then timing scripts (TIMERS)
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest $PYTESTSEL -x -q -p no:cacheprovider -s > gpurun_out/iter_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/iter_pytest.log
tail -8 gpurun_out/iter_pytest.log
for s in $TIMERS; do timeout 600 python $s 2>&1 | head -40; done
