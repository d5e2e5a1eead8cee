"""B200-native (sm_100a) PQL learner/actor hot path behind the reference's
Actor / V-learner / P-learner / replay-buffer interfaces."""
