# A/B of the K7 product: scratch/head (a saved build) vs $1 (default: the working tree's library), alternating
NEW=${1:-paper_1706_00241_b200/libdefcg_b200.so}
for r in 1 2 3; do
  DCG_LIB_PATH=scratch/head/libdefcg_b200.so python tools/k7_probe.py 50000 16 6 | sed 's/^/head /'
  DCG_LIB_PATH=$NEW python tools/k7_probe.py 50000 16 6 | sed 's/^/new  /'
done
