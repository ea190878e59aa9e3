cd $GRAFT_REPO_ROOT
for tps in 32 20 26 16 40 48; do
  SWEEP_TPP=16 SWEEP_LAYERS=21 SWEEP_LAYER=0 JENGA_DECODE_TILES_PER_SPLIT=$tps timeout 300 python profiles/sweep_decode.py --one 2>&1 | tail -1
done
for tpp in 32; do
  SWEEP_TPP=$tpp SWEEP_LAYERS=21 SWEEP_LAYER=0 timeout 300 python profiles/sweep_decode.py --one 2>&1 | tail -1
done
