# Static SASS mnemonic counts of the headline kernels (and the NEXT-4 ones) of libraid6c.so.
LIB=${1:-paper_cs_0611109_b200/libraid6c.so}
echo "# SASS evidence for $LIB (cuobjdump -sass): static mnemonic counts per kernel"
echo "# UBLKCP = cp.async.bulk (TMA bulk copy; .S.G = global->shared load, .G.S = shared->global store),"
echo "# SYNCS = mbarrier ops, SHF = funnel shifts, LOP3 = 3-input logic; no HMMA/UTC*MMA (no tensor cores)"
cuobjdump -sass "$LIB" > /tmp/sass_all.txt
for k in _ZN2zp9zp_kernelILi13ELi0ELb0EEEvNS_6ZpArgsE _ZN2zp9zp_kernelILi13ELi1ELb0EEEvNS_6ZpArgsE \
         _ZN2zp9zp_kernelILi59ELi4ELb0EEEvNS_6ZpArgsE _ZN2zp9zp_kernelILi59ELi5ELb0EEEvNS_6ZpArgsE; do
  echo "== $k ($(echo $k | c++filt))"
  awk -v k="$k" '/Function : /{f=($3==k)} f' /tmp/sass_all.txt | grep -oE '^\s+/\*[0-9a-f]+\*/\s+[A-Z][A-Z0-9._]+' | awk '{print $2}' | sort | uniq -c | sort -rn | grep -E "UBLK|SYNCS|SHF|LOP3|LDS|STS|FENCE|BAR|LDG|STG|RED"
done
echo "== tensor-core instructions in the whole library:"
grep -cE 'HMMA|UTC[A-Z]*MMA|HGMMA' /tmp/sass_all.txt
