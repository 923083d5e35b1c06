#!/bin/bash
# Mutation check for the oracle pins: copy the repository to a scratch
# directory, apply one sed edit to the COPY's oracle/oracle.c, run the copy's
# tests/test_oracle_pins.py.  The committed oracle is never touched.  Every
# mutation listed in DESIGN.md ("Oracle pins") must make at least one pin fail.
# usage: mutate_oracle.sh 'sed-expr'
set -e
SRC="$(cd "$(dirname "$0")/.." && pwd)"
SCR="$(mktemp -d /tmp/lmbp_mut.XXXXXX)"
trap 'rm -rf "$SCR"' EXIT
tar -C "$SRC" --exclude=.git --exclude=gpurun_out --exclude='*.so' --exclude=_obj --exclude=_variants -cf - . | tar -C "$SCR" -xf -
cd "$SCR"
cp oracle/oracle.c /tmp/lmbp_mut_orig.c
sed -i "$1" oracle/oracle.c
if cmp -s oracle/oracle.c /tmp/lmbp_mut_orig.c; then echo "NO CHANGE: $1"; fi
timeout 600 python -m pytest tests/test_oracle_pins.py -q -p no:cacheprovider 2>&1 | tail -1
