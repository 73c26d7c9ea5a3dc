set -u
bash tools/ablate.sh r01_v15 C3 "noob noob_s1 s1 noob_t256 noob_s1_t256 s1_t256" 0
