for i in 1 2; do
timeout 2400 python -m pytest -q -m gpu tests -p no:cacheprovider 2>&1 > /tmp/full.log; grep -E "passed|failed" /tmp/full.log | tail -1
grep -E "conservation|AssertionError: \[" /tmp/full.log | head -5
done
