export PYTHONPATH=.
for s in 64 65; do echo "c2 s=$s $(timeout 300 python scripts/time_cg64_c2.py c2 $s | tr '\n' ' ')"; done
timeout 300 python scripts/diag_i8.py gpurun_out/i8.npz 2>&1 | tail -3
