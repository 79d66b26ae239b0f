#!/bin/bash
# ncu --set full of the config-3 hot kernels of the final r02 build (tangent, residual, the GRID3
# matvec modes and k_update_xr), after a clean run of the same targets.
cd "$(dirname "$0")/.."
O=gpurun_out
export B200FEM_NO_GRAPH=1
python tools/ncu_targets.py all > $O/r02c_targets.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:'k_jacobian_v2|k_grid_pull' -c 2 \
    -o $O/r02c_ncu_tangent python tools/ncu_targets.py tangent > $O/r02c_ncu_tangent.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_residual' -c 2 \
    -o $O/r02c_ncu_residual python tools/ncu_targets.py residual > $O/r02c_ncu_residual.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_spmv_grid3|k_update_xr' -c 8 \
    -o $O/r02c_ncu_spmv python tools/ncu_targets.py spmv > $O/r02c_ncu_spmv.log 2>&1
for f in tangent residual spmv; do
  ncu -i $O/r02c_ncu_$f.ncu-rep --page raw --csv > $O/r02c_ncu_${f}_raw.csv 2>/dev/null
done
ls -la $O
