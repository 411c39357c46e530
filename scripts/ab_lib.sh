#!/bin/bash
# Same-box A/B of library builds on C2: LIBS="libtbsim_b200.so libtbsim_b200_x.so"
# (variant .so files built into the package directory; TBSIM_LIB selects one)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for rep in 1 2; do
  for lib in ${LIBS:-libtbsim_b200.so}; do
    TBSIM_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-traffic --no-c4 --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_ms']; print('$lib', round(d['value']), round(d['e2e']['value']), round(k['k_simulate'],3), round(k['k_sweep'],3))"
  done
done
