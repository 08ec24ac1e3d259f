#!/bin/bash
# every GPU test file in its own process (import-order independence), then the whole suite
for f in tests/test_*.py; do
  r=$(timeout 900 python -m pytest $f -m gpu -q 2>&1 | tail -1)
  echo "$f: $r"
done
