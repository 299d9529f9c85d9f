export PYTHONPATH=.
for nv in "" 2 20 100; do echo "E2E_NVML=$nv"; E2E_NVML=$nv timeout 300 python scripts/time_e2e_pipe.py tc_f16 2>&1 | tail -2; done
