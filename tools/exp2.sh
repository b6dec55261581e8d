timeout 900 python -m pytest tests -m gpu -q -x -k "bicgstab or batch or gmres or callable or krylov or streams or mutated" 2>&1 | tail -2
