set -e
cd $GRAFT_REPO_ROOT
for k in 4 8 2; do
  NVCC_EXTRA="-DSINCOS_NUDFT_KPT=$k" python -c "
import os, subprocess, sys
sys.path.insert(0, '.')
from paper_cs_0406049_b200 import _build
cmd=[_build.nvcc(), *_build.NVCC_FLAGS, '-DSINCOS_NUDFT_KPT=$k', '-o', _build.LIB, *_build.sources()]
subprocess.check_call(cmd, cwd=_build.PKG)
"
  echo "KPT=$k"; python tools/time_nudft.py; python tools/time_nudft.py
done
