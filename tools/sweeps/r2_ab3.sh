L=paper_2402_01181_b200
for r in 1 2; do
ROUNDS=1 bash tools/sweeps/ab.sh base=$L/libsoftmpm_b200.so 2>&1 | grep -v '^ \|Trace\|json'
SOFTMPM_PDL=1 ROUNDS=1 bash tools/sweeps/ab.sh pdl=$L/libsoftmpm_b200.so 2>&1 | grep -v '^ \|Trace\|json'
SOFTMPM_MEGA=1 ROUNDS=1 bash tools/sweeps/ab.sh mega=$L/libsoftmpm_b200.so 2>&1 | grep -v '^ \|Trace\|json'
SOFTMPM_GRIDOP_SIMPLE=0 ROUNDS=1 bash tools/sweeps/ab.sh oldgrid=$L/libsoftmpm_b200.so 2>&1 | grep -v '^ \|Trace\|json'
done
for c in c4 c5; do
CONFIG=$c ROUNDS=1 STEPS=4 bash tools/sweeps/ab.sh base_$c=$L/libsoftmpm_b200.so 2>&1 | grep -v '^ \|Trace\|json'
SOFTMPM_PDL=1 CONFIG=$c ROUNDS=1 STEPS=4 bash tools/sweeps/ab.sh pdl_$c=$L/libsoftmpm_b200.so 2>&1 | grep -v '^ \|Trace\|json'
done
