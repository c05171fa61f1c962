#!/bin/bash
# verify_plan wall time on 405B for env variants, alternating, same box.
# Usage: bash scripts/e2e_ab.sh "ENV=.." "ENV=.." ...
for r in 1 2; do
  for v in "$@"; do
    echo "== $v"
    env $v timeout 600 python scripts/e2e_breakdown.py llama3-405b-tp8pp16dp2 2>/dev/null | grep "^verify_plan" | tail -6 | awk '{print $2}' | tr '\n' ' '; echo
  done
done
