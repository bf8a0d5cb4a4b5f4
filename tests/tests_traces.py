"""Hand-traced scripted requests (SURVEY §8(c) traces A and B) shared by CPU and GPU tests."""
import numpy as np

from synth import Request, Script


def trace_A_request(rid=0):
    scores = np.zeros((4, 4), np.float32)
    scores[:, 0] = [0.6, 0.4, 0.3, 0.45]
    scores[0, 1], scores[3, 1] = 0.55, 0.2
    scores[3, 2] = 0.6
    sc = Script(np.array([40, 20, 64, 50], np.int32), scores, np.array([0.7, 0, 0, 0], np.float32),
                np.zeros(4, np.int32))
    return Request(rid, np.arange(2, 5, dtype=np.int32), 4, 2, float(np.float32(0.5)), 2, sc)


def trace_B_request(rid=0):
    sc = Script(np.array([30, 10, 50, 25], np.int32), np.zeros((4, 4), np.float32), np.full(4, 0.5, np.float32),
                np.zeros(4, np.int32))
    return Request(rid, np.arange(2, 19, dtype=np.int32), 4, 2, -1.0, 0, sc)
