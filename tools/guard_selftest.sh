#!/bin/bash
# The debug build's guard bands catch an overrun: a throw-away build with one
# injected write past the MSF key array must fail kdb_mst with KDB_EINTERNAL.
set -u
NCCL_INC=$(python -c "import os,nvidia.nccl as m; print(os.path.join(list(m.__path__)[0],'include'))")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -Iinclude -I$NCCL_INC \
  --expt-relaxed-constexpr -DKDB_GUARDS=1 -DKDB_INJECT_OVERRUN=1 -o /tmp/libkdb_inject.so \
  paper_2009_04552_b200/csrc/kdb.cu -ldl || exit 2
KDB_LIBRARY=/tmp/libkdb_inject.so python tools/debug_cases.py c1 > /tmp/inject.log 2>&1
rc=$?
grep -o "KDB_EINTERNAL.*guard band[^\"]*" /tmp/inject.log | head -1
echo "injected overrun run rc=$rc (non-zero expected)"
[ $rc -ne 0 ] && grep -q "guard band" /tmp/inject.log && echo "guard self-test: PASS" || echo "guard self-test: FAIL"
