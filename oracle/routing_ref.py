"""Oracle restatement of moekit/trace.py statistics and moekit/placement.py
(TEST INFRASTRUCTURE ONLY).

A trace is represented as an int array ``paths[events, layers, top_k]`` with
ascending expert ids per layer (the RoutingEvent.path invariant,
trace.py:40-44 / 82-85).
"""

from __future__ import annotations

from collections import Counter

import numpy as np


def expert_freq(paths: np.ndarray, experts: int) -> np.ndarray:
    """trace.expert_freq (trace.py:216-225): counts[layer, expert]."""
    paths = np.asarray(paths)
    if paths.shape[0] == 0:
        raise ValueError("empty trace")
    ev, layers, k = paths.shape
    counts = np.zeros((layers, experts), dtype=np.int64)
    for layer in range(layers):
        counts[layer] = np.bincount(paths[:, layer, :].ravel(), minlength=experts)
    return counts


def path_stats(paths: np.ndarray):
    """trace.path_stats (trace.py:207-213): [(path, count)] by descending
    count, ties by ascending path (tuple order)."""
    paths = np.asarray(paths)
    if paths.shape[0] == 0:
        raise ValueError("empty trace")
    keys = [tuple(tuple(int(e) for e in sel) for sel in p) for p in paths]
    return sorted(Counter(keys).items(), key=lambda kv: (-kv[1], kv[0]))


def plan_frequency(counts: np.ndarray, budget: int):
    """placement.plan_frequency (placement.py:75-93)."""
    layers, experts = counts.shape
    if not 0 <= budget <= layers * experts:
        raise ValueError("bad budget")
    order = sorted((-int(counts[l, e]), l, e) for l in range(layers) for e in range(experts))
    res = [set() for _ in range(layers)]
    for _, l, e in order[:budget]:
        res[l].add(e)
    return [frozenset(r) for r in res]


def plan_path(entries, layers: int, experts: int, budget: int):
    """placement.plan_path (placement.py:96-121): whole paths until the next
    one does not fit."""
    if not 0 <= budget <= layers * experts:
        raise ValueError("bad budget")
    res = [set() for _ in range(layers)]
    used = 0
    for path, _ in entries:
        new = [(l, e) for l, sel in enumerate(path) for e in sel if e not in res[l]]
        if used + len(new) > budget:
            break
        for l, e in new:
            res[l].add(e)
        used += len(new)
    return [frozenset(r) for r in res]


def plan_two_stage(entries, counts: np.ndarray, top_k_per_layer: int, supplement: int):
    """placement.plan_two_stage (placement.py:124-176): per-layer path fill,
    then per-layer frequency supplement (ties to the lower id)."""
    layers, experts = counts.shape
    per_layer = top_k_per_layer + supplement
    if top_k_per_layer < 0 or supplement < 0 or per_layer > experts:
        raise ValueError("bad per-layer counts")
    res = [set() for _ in range(layers)]
    for path, _ in entries:
        if all(len(r) >= top_k_per_layer for r in res):
            break
        for l, sel in enumerate(path):
            for e in sorted(sel):
                if len(res[l]) >= top_k_per_layer:
                    break
                res[l].add(e)
    for l in range(layers):
        ranked = sorted(range(experts), key=lambda e: (-int(counts[l, e]), e))
        for e in ranked:
            if len(res[l]) >= per_layer:
                break
            res[l].add(e)
    return [frozenset(r) for r in res]


def evaluate_plan(residents, paths: np.ndarray, top_k: int):
    """placement.evaluate_plan (placement.py:178-208) -> (per_layer, mean,
    std, gap)."""
    paths = np.asarray(paths)
    layers = len(residents)
    if paths.shape[0] == 0 or layers == 0:
        return np.zeros(layers), 0.0, 0.0, 0.0
    hits = np.zeros(layers, dtype=np.int64)
    for l in range(layers):
        mask = np.isin(paths[:, l, :], np.array(sorted(residents[l]), dtype=paths.dtype))
        hits[l] = int(mask.sum())
    per = hits / float(top_k * paths.shape[0])
    return per, float(per.mean()), float(per.std()), float(per.max() - per.min())
