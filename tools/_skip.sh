python tools/skip_probe.py actor 6
timeout 300 python tools/ab_actor.py 2>&1 | grep "N=16384 algo=0"
timeout 900 python -m pytest tests -m gpu -x -q -k "actor or sac or plearner or vlearner or precision or dropin" 2>&1 | tail -3
