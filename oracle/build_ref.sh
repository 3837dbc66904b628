#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY.  Builds the reference's own compiled screening core
# (`pkg/src/ltllearn/_speedups.pyx`, Cython -> C++) from the sources WHERE THEY LIE under
# /root/reference into oracle/_ref/ (git-ignored, shipped to the GPU box by gpurun).
# Nothing from the reference is copied into the repo: the generated C / C++ lives in a temp dir
# and only shared objects are kept.  The reference's Python modules around the core (enumerator,
# cache, bitsem, formula, kernels, traces, dnc, benchgen, oracle, _kernels_py) are compiled the same
# way (Cython -> gcc, binaries only), so that on the GPU box -- where /root/reference does not
# exist -- tests can run the reference's OWN `enum_learn` with the CUDA core plugged into
# `kernels.make_core` (tests/test_gpu_reference_driven.py) and bench.py can time the reference's own
# learner inside its limits.
set -euo pipefail
REF=${LTL_REFERENCE_ROOT:-/root/reference}
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
OUT="$HERE/_ref/ltllearn"
SRC="$REF/pkg/src/ltllearn/_speedups.pyx"
if [ ! -f "$SRC" ]; then
  echo "build_ref: $SRC not present (GPU box?) - keeping whatever is prebuilt" >&2
  exit 0
fi
PY=${PYTHON:-python}
mkdir -p "$OUT"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
"$PY" -m cython --cplus -3 --module-name ltllearn._speedups -o "$TMP/_speedups.cpp" "$SRC"
EXT=$("$PY" -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
INC=$("$PY" -c "import sysconfig; print(sysconfig.get_paths()['include'])")
g++ -O3 -std=c++17 -shared -fPIC -w -I"$INC" "$TMP/_speedups.cpp" -o "$OUT/_speedups$EXT"
rm -f "$OUT/_kernels_py.py"  # (older builds generated a stand-in for the one name the compiled core imports)
for m in _kernels_py kernels bitsem formula traces cache enumerator dnc benchgen oracle; do
  "$PY" -m cython -3 --module-name "ltllearn.$m" -o "$TMP/$m.c" "$REF/pkg/src/ltllearn/$m.py" > /dev/null
  gcc -O2 -shared -fPIC -w -I"$INC" "$TMP/$m.c" -o "$OUT/$m$EXT"
done
echo "build_ref: built $OUT/_speedups$EXT"
