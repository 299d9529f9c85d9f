export PYTHONPATH=.
mkdir -p gpurun_out
timeout 300 python scripts/time_e2e_upload.py tc_f16 1 > gpurun_out/zc_plain.log 2>&1 || exit 1
tail -3 gpurun_out/zc_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/zc_launches.csv python scripts/time_e2e_upload.py tc_f16 1 > gpurun_out/zc_ncu.log 2>&1
wc -l gpurun_out/zc_launches.csv
