#!/bin/bash
# Boundary proof: run the reference's OWN tests (tests/test_energy.py,
# tests/test_detect.py) with diffwatt.energy and diffwatt.detect resolved to
# this package.  Two halves, because /root/reference exists only in the build
# container and the GPU only on the gpurun box:
#   bash scripts/ref_tests_shim.sh make   (here)  copies the reference package
#        and tests into the git-ignored _refshim/ (never committed) and swaps
#        the two modules for re-exports of paper_2512_08365_b200.{energy,detect};
#   bash scripts/ref_tests_shim.sh run    (GPU box) runs the tests there;
#   bash scripts/ref_tests_shim.sh clean  (here)  removes _refshim/.
set -e
D=_refshim
case "$1" in
make)
  R=/root/reference/pkg
  rm -rf $D; mkdir -p $D
  cp -r $R/src/diffwatt $D/diffwatt; cp -r $R/tests $D/tests
  for m in energy detect; do
    printf 'import sys\nimport paper_2512_08365_b200.%s as _impl\nsys.modules[__name__] = _impl\n' $m > $D/diffwatt/$m.py
  done ;;
run)
  mkdir -p gpurun_out
  (cd $D && PYTHONPATH=$GRAFT_REPO_ROOT:$PWD timeout 1200 python -m pytest tests/test_energy.py tests/test_detect.py \
      -q -p no:cacheprovider -rA 2>&1) > gpurun_out/ref_tests.log; echo "ref tests rc=$?"
  python - <<'PY'
import sys; sys.path.insert(0, "."); sys.path.insert(0, "_refshim")
import diffwatt.energy, diffwatt.detect, paper_2512_08365_b200 as p
assert diffwatt.energy is p.energy and diffwatt.detect is p.detect
print("shim check: diffwatt.energy ->", diffwatt.energy.__file__, "| diffwatt.detect ->", diffwatt.detect.__file__)
PY
  tail -5 gpurun_out/ref_tests.log ;;
clean) rm -rf $D ;;
esac
