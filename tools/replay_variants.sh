# replay probes for library variants: bash tools/replay_variants.sh lib1.so lib2.so ...
for lib in "$@"; do
  for a in "1000000 8 8 3 knn" "10000000 64 8 3 synthetic" "10000000 64 8 3 knn"; do
    NOMAD_B200_LIB=$PWD/$lib timeout 400 python tools/replay_probe.py $a 2>&1 | tail -1 | sed "s|^|$(basename $lib) |"
  done
  NOMAD_B200_LIB=$PWD/$lib timeout 300 python tools/replay_chain.py 400000 8 2 | sed "s|^|$(basename $lib) |"
done
