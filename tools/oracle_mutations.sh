#!/bin/bash
# Mutation check of the oracle pins (VERDICT r1 "What's weak" 1): applies each plausible mistake
# to a scratch copy of oracle/ and runs the oracle pin tests; every mutation must fail a pin.
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
W=$(mktemp -d)
cp -r "$ROOT"/{oracle,scenes,tests,pytest.ini} "$W"/
cd "$W"
run() { python -m pytest tests/test_oracle_pins_r2.py tests/test_oracle_contact.py tests/test_oracle_solve.py -q -p no:cacheprovider 2>&1 | tail -1; }
restore() { cp "$ROOT"/oracle/*.py oracle/; }
echo "M0 (unmutated):"; run
sed -i 's/lam = np.maximum(lam, 0.0)/lam = np.abs(lam)/' oracle/barrier.py
echo "M1 psd_project |lambda|:"; run; restore
sed -i 's/dof = (3 \* ids\[:, :, None\]/dof = (3 * ids[:, ::-1, None]/' oracle/contact.py
echo "M2 pull-back stencil reversed:"; run; restore
sed -i 's|alpha = alpha / 2.0|alpha = alpha / 3.0|' oracle/solver.py
echo "M3a line search halves by 3:"; run; restore
sed -i 's|for h in range(self.ls_max_halvings + 1):|for h in range(3):|' oracle/solver.py
echo "M3b line search cap of 2 halvings:"; run; restore
sed -i 's/lp_, hp_ = lo - dh, hi + dh/lp_, hp_ = lo, hi/; s/lt = lo\[tris\].min(axis=1) - dh/lt = lo[tris].min(axis=1)/; s/ht = hi\[tris\].max(axis=1) + dh/ht = hi[tris].max(axis=1)/; s/le = lo\[edges\].min(axis=1) - dh/le = lo[edges].min(axis=1)/; s/he = hi\[edges\].max(axis=1) + dh/he = hi[edges].max(axis=1)/' oracle/ccd.py
echo "M4 swept boxes without d_hat inflation:"; run; restore
rm -rf "$W"
