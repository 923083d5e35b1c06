#!/bin/bash
# Mutation check for the oracle pins: apply one sed edit to oracle/oracle.c,
# run tests/test_oracle_pins.py, restore.  Every mutation listed in DESIGN.md
# ("Oracle pins") must make at least one pin fail.
# usage: run.sh 'sed-expr'
cd "$(dirname "$0")/.."
mkdir -p /tmp/mut
git diff --quiet HEAD -- oracle/oracle.c || { echo "oracle/oracle.c differs from HEAD; refusing"; exit 1; }
cp oracle/oracle.c /tmp/mut/orig.c
trap 'cp /tmp/mut/orig.c oracle/oracle.c; rm -f oracle/liboracle.so' EXIT
sed -i "$1" oracle/oracle.c
if cmp -s oracle/oracle.c /tmp/mut/orig.c; then echo "NO CHANGE: $1"; fi
rm -f oracle/liboracle.so
timeout 600 python -m pytest tests/test_oracle_pins.py -q 2>&1 | tail -1
cp /tmp/mut/orig.c oracle/oracle.c
rm -f oracle/liboracle.so
