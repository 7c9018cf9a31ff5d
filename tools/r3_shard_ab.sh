for L in tools/libpmh_head.so paper_1911_00675_b200/libpmh.so tools/libpmh_sn1.so; do
  echo "== $L"
  for a in probminhash1 probminhash2 probminhash3 probminhash4; do PMH_LIB_PATH=$PWD/$L python tools/shard_classes.py $a 8 2>&1 | head -1; done
  PMH_LIB_PATH=$PWD/$L python tools/shard_sim.py 1,8 --concurrent 2>&1 | cut -c1-120
done
