# A/B of compile-time variants built locally into paper_2512_19925_b200/_build_<name>
rm -f gpurun_out/ab_summary.txt
for c in ${CFGS:-c5 c2}; do
  for n in base "$@"; do
    if [ "$n" = base ]; then L=""; else L="HWWG_LIB=paper_2512_19925_b200/_build_$n/libhwwg.so"; fi
    CFG=$c bash scripts/gpu_ab.sh "$L HWWG_TAG=$c/$n" > /dev/null 2>&1
  done
done
