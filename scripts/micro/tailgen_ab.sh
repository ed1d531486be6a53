# record: the SPO_CELL_TAILS_GENERAL variant was built for this A/B only (profiles/r02/v_cell_groups.md); not in the sources
# aligned V groups: a cell's 1..VGROUP-1 position tail groups on the general loop (-DSPO_CELL_TAILS_GENERAL=1,
# libspo_b200_tailgen.so) against one unrolled same-cell body per size (default build)
P=$PWD/paper_1611_02665_b200
for lib in default tailgen; do
  if [ $lib = default ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_$lib.so; fi
  for vg in 3 4; do
    echo "== lib $lib VGROUP $vg"
    SPO_VGROUP=$vg timeout 600 python scripts/micro/env_ab.py --envs "SPO_VCELL=0;SPO_VCELL=1" \
      --cases cfg5-v,cfg5-v-6144w,cfg4-v-8192w,cfg4-v-16384w 2>&1 | grep '^{'
  done
done
unset SPO_LIB
