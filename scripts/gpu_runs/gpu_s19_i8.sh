export PYTHONPATH=.
timeout 300 python scripts/diag_i8.py gpurun_out/i8.npz 2>&1 | tail -10
timeout 300 python scripts/time_cg64_c2.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hv_i8 -c 3 --csv python scripts/time_cg64_c2.py 2>/dev/null | grep hv_i8 | tail -1
