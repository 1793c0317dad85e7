bash tools/quick.sh
CACHE=none bash tools/prof_launches.sh ${1:-w}
