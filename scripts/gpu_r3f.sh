#!/bin/bash
set -u
for bb in 400 600 800 1200; do
  echo "== PQW_BUNDLE_BASE=$bb"
  PQW_BUNDLE_BASE=$bb timeout 900 python scripts/per_program_time.py llama3-405b-tp8pp16dp2 2>&1 | head -12
done
