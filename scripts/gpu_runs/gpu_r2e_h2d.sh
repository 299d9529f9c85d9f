# e2e: two-stream H2D experiment, and the effect of an NVML sampler thread
export PYTHONPATH=.
timeout 300 python scripts/time_e2e_pipe.py tc_f16 "1;;|2;0.68,0.32;0.68,0.32|2" 2>&1 | tail -5
E2E_NVML=2 timeout 300 python scripts/time_e2e_pipe.py tc_f16 "1;" 2>&1 | tail -2
E2E_NVML=50 timeout 300 python scripts/time_e2e_pipe.py tc_f16 "1;" 2>&1 | tail -2
