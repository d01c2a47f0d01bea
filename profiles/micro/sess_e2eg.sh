set -x
for i in 1 2; do timeout 300 python profiles/micro/time_run_e2e.py; done
