# wgp_hv row-chunk pipeline: test + e2e timing variants (config 1)
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host_row_chunks or config1 or hv_impls or row_sharding" 2>&1 | tail -4
for r in 1 2; do
for pipe in 1 0.72,0.28 0.5,0.5 0.8,0.2 0.65,0.35 0.55,0.3,0.15; do
  WGP_HV_PIPE=$pipe timeout 120 python scripts/time_e2e_pipe.py tc_f16 2>&1 | tail -1
done; done
WGP_HV_PIPE=1 timeout 120 python scripts/time_e2e_pipe.py tc 2>&1 | tail -1
timeout 120 python scripts/time_e2e_pipe.py tc 2>&1 | tail -1
