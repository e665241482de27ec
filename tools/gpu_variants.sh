for v in r0_s1 r1_s1 r0_s0 r1_s0; do
  FASTRON_LIB=build/variants/lib_$v.so timeout 300 python tools/variant_check.py 2>&1 | tail -1
done
