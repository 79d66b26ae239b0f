for i in 1 2; do
  for v in "" 30 15 60; do
    if [ -z "$v" ]; then unset B200FEM_GRID_SLAB; else export B200FEM_GRID_SLAB=$v; fi
    python tools/krylov_profile.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['slab']='$v' or 'plain'; print(json.dumps(d))" >> gpurun_out/r02_slab_jacobi_ab.jsonl
  done
done
unset B200FEM_GRID_SLAB
timeout 900 python tools/newton_ab.py B200FEM_GRID_SLAB=30 >> gpurun_out/r02_slab_jacobi_ab.jsonl 2>/dev/null
cat gpurun_out/r02_slab_jacobi_ab.jsonl | cut -c1-400
