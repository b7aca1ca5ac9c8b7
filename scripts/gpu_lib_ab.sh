# A/B of library builds: for every build_ab/lib_<tag>.so, swap it in and run the small/mid-N probe.
# usage (GPU box): bash scripts/gpu_lib_ab.sh "<N list>" [precision]
LIB=paper_1907_04839_b200/liblmshoot_b200.so
cp $LIB /tmp/lib_orig.so
for f in build_ab/lib_*.so; do
  cp $f $LIB
  echo "== $f"
  for n in $1; do python scripts/gpu_small_n.py $n ${2:-f32}; done
done
cp /tmp/lib_orig.so $LIB
