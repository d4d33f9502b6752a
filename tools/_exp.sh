tools/ab.sh "L8 L12 L16" 1 --batch 8
tools/ab.sh "L8 L12 L16" 1 --batch 4
