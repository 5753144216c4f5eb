#!/bin/bash
# Source-level ncu capture of ONE H-Cholesky launch (k_exec_rq, whole GPU, n = 64k mesh):
# per-source-line stall samples / instructions / shared-memory bank conflicts, exported as CSV.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
cat > /tmp/one_chol.py << 'PY'
import sys
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import perturbed_mesh
pts = perturbed_mesh(256, 0.4, 2)
H = hm.HMatrix(pts, (1.0, 0.1, 0.5), eps=1e-7, leaf=64, eta=2.0, kmax=64)
H.cholesky()
print("ok")
PY
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_exec_rq -s 1 -c 1 \
  -o gpurun_out/chol_src python /tmp/one_chol.py > gpurun_out/ncu_src.log 2>&1
echo "capture rc=$?"
ncu -i gpurun_out/chol_src.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/chol_src_sass.csv 2>/dev/null
ncu -i gpurun_out/chol_src.ncu-rep --page source --csv --print-source cuda > gpurun_out/chol_src_cuda.csv 2>/dev/null
ncu -i gpurun_out/chol_src.ncu-rep --page raw --csv > gpurun_out/chol_src_raw.csv 2>/dev/null
ls -la gpurun_out/chol_src*
rm -f gpurun_out/chol_src.ncu-rep
