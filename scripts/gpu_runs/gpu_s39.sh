export PYTHONPATH=.
for s in 64 65 17; do echo "c2 s=$s $(timeout 300 python scripts/time_cg64_c2.py c2 $s | tr '\n' ' ')"; done
echo "c4 s=65 i8 $(timeout 900 python scripts/time_cg64_c2.py c4 65 | tr '\n' ' ')"
