# wgp_hv row-chunk pipeline sweep + zero-copy input (config 1, tc_f16)
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host_row_chunks" 2>&1 | tail -2
for zc in 0 1; do
for pipe in 1 0.6,0.4 0.62,0.38 0.65,0.35 0.68,0.32 0.7,0.3 0.5,0.3,0.2 0.45,0.3,0.25 0.4,0.35,0.25 0.5,0.25,0.25; do
  WGP_HV_ZC=$zc WGP_HV_PIPE=$pipe timeout 120 python scripts/time_e2e_pipe.py tc_f16 2>&1 | tail -1 | sed "s/^/zc=$zc /"
done; done
WGP_HV_ZC=1 WGP_HV_PIPE=0.65,0.35 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host_row_chunks or config1 or hv_impls" 2>&1 | tail -2
