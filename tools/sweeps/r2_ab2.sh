L=paper_2402_01181_b200
for r in 1 2; do
ROUNDS=1 bash tools/sweeps/ab.sh base=$L/libsoftmpm_b200.so seg2=$L/libsoftmpm_b200_seg2.so seg8=$L/libsoftmpm_b200_seg8.so 2>&1 | grep -v '^ \|Trace\|json'
for ips in 3 6 8; do SOFTMPM_ITEMS_PER_SM=$ips ROUNDS=1 bash tools/sweeps/ab.sh ips$ips=$L/libsoftmpm_b200.so 2>&1 | grep -v '^ \|Trace\|json'; done
done
