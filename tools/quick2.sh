# GPU tests, short bench, launch list
tag=${1:-q}
bash tools/quick.sh
bash tools/prof_launches.sh $tag
