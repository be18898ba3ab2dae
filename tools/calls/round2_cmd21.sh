bash tools/ab.sh 5 col256 col256g2
bash tools/ab.sh 2 col256 col256g2
bash tools/ab.sh 5 col256
