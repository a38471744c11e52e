for lib in paper_1208_0945_b200/_lib/libbsccs_b200*.so; do echo "== $lib"; for w in "1M" "10M"; do BSCCS_B200_LIB=$PWD/$lib timeout 200 python scripts/probe_fit.py $w; done; done
# A/B of k_ccd kernel shapes (threads x register tiles) on one probe
