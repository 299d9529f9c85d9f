for impl in ${IMPLS:-tc tc_f16}; do for dbg in ${DBGS:-0}; do echo "impl=$impl dbg=$dbg"; WGP_TC_DEBUG=$dbg timeout 60 python scripts/diag_f16_time.py $impl 2>&1 | tail -1; done; done
