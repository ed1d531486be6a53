# record: the SPO_CELL_RT variant lived in commit be5f965 only (removed after this A/B, profiles/r02/v_cell_groups.md)
# aligned V groups: one unrolled body per group size (default build) against one body with
# the size tested per position (-DSPO_CELL_RT=1, libspo_b200_cellrt.so), group sizes swept;
# SPO_VCELL=0 (fixed groups) rides along as the reference and the bitwise check
P=$PWD/paper_1611_02665_b200
for lib in default cellrt; do
  if [ $lib = default ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_$lib.so; fi
  for vg in 3 4 5; do
    echo "== lib $lib VGROUP $vg"
    SPO_VGROUP=$vg timeout 900 python scripts/micro/env_ab.py --envs "SPO_VCELL=0;SPO_VCELL=1" \
      --cases cfg5-v,cfg5-v-6144w,cfg4-v-8192w,cfg4-v-12288w,cfg4-v-16384w 2>&1 | grep '^{'
  done
done
unset SPO_LIB
