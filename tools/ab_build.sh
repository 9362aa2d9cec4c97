# Build the current sources into lib/ab/<name>/libhmx_gpu.so (A/B experiments:
# run with HMX_GPU_LIB=paper_1911_00093_b200/lib/ab/<name>/libhmx_gpu.so)
name=$1
out=paper_1911_00093_b200/lib/ab/$name
mkdir -p $out
python - <<PY
import sys, shutil
sys.path.insert(0, '.')
from paper_1911_00093_b200 import _native
lib = _native.build_gpu(force=True)
shutil.copy(lib, '$out/libhmx_gpu.so')
print('built', '$out')
PY
