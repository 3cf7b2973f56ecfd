for v in "16 3" "32 2" "16 4" "32 3"; do set -- $v
  rm -f build/gemm_f64.o paper_2605_16058_b200/libstarm.so; make -j8 NVEXTRA="-DGEMM_BK=$1 -DGEMM_STAGES=$2" > /dev/null 2>&1
  echo "BK=$1 STAGES=$2: $(python scripts/run_gemm.py)"
done
