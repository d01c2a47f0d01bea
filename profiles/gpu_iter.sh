# one GPU iteration: targeted tests, then timings (args: pytest selection)
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest $PYTESTSEL -x -q -p no:cacheprovider -s > gpurun_out/iter_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/iter_pytest.log
tail -5 gpurun_out/iter_pytest.log
grep "fig6" gpurun_out/iter_pytest.log
for s in $TIMERS; do timeout 300 python $s 2>&1 | tail -3; done
