export PYTHONPATH=.
for l in lib_full lib_nomma lib_nomath; do for s in 64 65; do
  t=$(WGP_LIBRARY=$PWD/ab/$l.so timeout 300 ncu --metrics gpu__time_duration.sum -k regex:hv_i8_kernel -s 1 -c 2 --csv python scripts/time_hv64_kernel.py $s 2>/dev/null | grep hv_i8 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')
  echo "$l s=$s kernel_ns: $t"
done; done
