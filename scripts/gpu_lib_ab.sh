# A/B of library builds: for every build_ab/lib_<tag>.so, swap it in and run a probe.
# usage (GPU box): bash scripts/gpu_lib_ab.sh "<command with its own args>"
LIB=paper_1907_04839_b200/liblmshoot_b200.so
cp $LIB /tmp/lib_orig.so
for f in build_ab/lib_*.so; do
  cp $f $LIB
  echo "== $f"
  eval "$1"
done
cp /tmp/lib_orig.so $LIB
