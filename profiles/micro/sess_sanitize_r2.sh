set -x
for w in xp km codec replay; do
  timeout 900 compute-sanitizer --tool memcheck --leak-check no --print-limit 5 python profiles/micro/sanitize_r2.py $w 2>&1 | tail -3
done
for w in km codec; do
  timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python profiles/micro/sanitize_r2.py $w 2>&1 | tail -3
done
