export PYTHONPATH=.
for mode in "" 1; do
for i in 1 2; do
echo "WGP_HV_PIPE=$mode"
WGP_HV_PIPE=$mode WGP_HV_PLAN_DEBUG=1 timeout 300 python bench.py --no-outer --no-large --no-cpu-baseline 2>&1 >/dev/null | grep -v "plan" | tail -2
done; done
timeout 300 python scripts/time_e2e_pipe.py tc_f16 2>&1 | tail -2
