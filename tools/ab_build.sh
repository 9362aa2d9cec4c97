# Build the current sources into lib/ab/<name>/libhmx_gpu.so (A/B experiments:
# run with HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/<name>/libhmx_gpu.so).
# The in-tree lib/libhmx_gpu.so is restored afterwards.
name=$1
out=paper_1911_00093_b200/lib/ab/$name
main=paper_1911_00093_b200/lib/libhmx_gpu.so
mkdir -p $out
[ -f $main ] && cp -p $main /tmp/libhmx_gpu.so.keep.$$
python - <<PY
import sys, shutil
sys.path.insert(0, '.')
from paper_1911_00093_b200 import _native
lib = _native.build_gpu(force=True)
shutil.copy(lib, '$out/libhmx_gpu.so')
print('built', '$out')
PY
if [ -f /tmp/libhmx_gpu.so.keep.$$ ]; then cp -p /tmp/libhmx_gpu.so.keep.$$ $main; rm -f /tmp/libhmx_gpu.so.keep.$$; fi
