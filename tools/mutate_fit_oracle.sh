#!/bin/bash
# Mutation check for the fitter-oracle pins: apply one python-level text
# substitution to oracle/fit.py, run tests/test_fit_oracle.py, restore.
# Every mutation below must make at least one pin fail.
# Runs in a scratch copy of the repository: the committed oracle/fit.py is
# never edited (a mutant once reached a commit when this edited in place).
SRC="$(cd "$(dirname "$0")/.." && pwd)"
SCR="$(mktemp -d /tmp/lmbp_fitmut.XXXXXX)"
trap 'rm -rf "$SCR"' EXIT
tar -C "$SRC" --exclude=.git --exclude=gpurun_out --exclude='*.so' --exclude=_obj --exclude=_variants -cf - . | tar -C "$SCR" -xf -
cd "$SCR"
cp oracle/fit.py /tmp/lmbp_fit_orig.py
run() {
  python - "$1" "$2" <<'PY'
import sys
p = "oracle/fit.py"; s = open(p).read()
old, new = sys.argv[1], sys.argv[2]
assert old in s, old
open(p, "w").write(s.replace(old, new, 1))
PY
  echo "== $1  ->  $2"
  timeout 900 python -m pytest tests/test_fit_oracle.py -q -x 2>&1 | tail -1
  cp /tmp/lmbp_fit_orig.py oracle/fit.py
}
run 'math.sqrt(-2.0 * math.log(eps))' 'math.sqrt(-math.log(eps))'                       # GELU tail bound
run '-2.0 * math.log(eps / 2.0)' '-2.0 * math.log(eps)'                                 # SiLU tail bound
run '[1.0 - a.sum()]' '[a.sum()]'                                                       # last weight
run 'max(x - ci, 0.0)' 'max(ci - x, 0.0)'                                               # ReLU direction
run 'if x > ci' 'if x < ci'                                                             # step direction
run '(act(kind, x) - combo(x, w, c)) ** 2' 'abs(act(kind, x) - combo(x, w, c))'        # square dropped
run '(act_deriv(kind, x) - combo_deriv(x, w, c)) ** 2' '(act(kind, x) - combo_deriv(x, w, c)) ** 2'  # h for h'
run 'theta[m - 1:].copy()' 'theta[m - 2:-1].copy()'                                     # threshold slice
run 'levels = np.concatenate([[0.0], np.cumsum(ws)])' 'levels = np.concatenate([np.cumsum(ws), [1.0]])'  # levels
