#!/bin/bash
# SASS evidence for the hot kernels (run here, no GPU needed): instruction
# classes that prove TMA (UTMALDG / UBLKCP), tcgen05 (UTCHMMA, LDTM/STTM,
# UTCBAR), CTA pairs (.2CTA), mbarrier pipelines (SYNCS) and the mma.sync
# decode math (HMMA / LDSM / MOVM), per object of the product library.
cd "$(dirname "$0")/.."
for o in decode_tc prefill_tc5 cache_write decode tables; do
  echo "== build/jenga_b200/$o.cu.o"
  cuobjdump -sass build/jenga_b200/$o.cu.o | grep -oE "(UTMALDG[.A-Z0-9]*|UBLKCP[.A-Z.]*|UTCHMMA[.A-Z0-9]*|UTCBAR[.A-Z0-9]*|LDTM[.A-Z0-9]*|STTM[.A-Z0-9]*|HMMA\.[0-9A-Z.]*|LDSM[.A-Z0-9]*|MOVM[.A-Z0-9]*|SYNCS[.A-Z0-9]*|MUFU\.[A-Z0-9]*|UTCATOMSWS[.A-Z0-9]*)" | sort | uniq -c | sort -rn
  echo "-- kernels:"
  cuobjdump -sass build/jenga_b200/$o.cu.o | grep -oE "Function : [A-Za-z0-9_]+" | sort -u | sed 's/Function : /   /' | c++filt | cut -c1-160
done
