set -u
bash tools/ablate.sh r01_v50 C3 "t768 tile256 chunk2048 taildiv16" 0
