"""Table 1 of the paper (table `model_config`).

"The latency is measured for a single query with a sequence length of 2048
on a single GPU. BERT-104B's latency is reported using a minimal degree of
inter-op parallelism.".  Usable memory per 16 GB V100 is "around
13GB" (P:106 footnote).
"""

GB = 10**9
MS = 10**6  # ns per millisecond

# name -> (weight bytes, single-GPU latency ns)
MODELS = {
    "BERT-1.3B": (int(2.4 * GB), 151 * MS),
    "BERT-2.7B": (int(5.4 * GB), 238 * MS),
    "BERT-6.7B": (int(13.4 * GB), 395 * MS),
    "BERT-104B": (int(208 * GB), 4600 * MS),
    "MoE-1.3B": (int(2.6 * GB), 150 * MS),
    "MoE-2.4B": (int(4.8 * GB), 171 * MS),
    "MoE-5.3B": (int(10.6 * GB), 234 * MS),
}

# model-set instance counts, columns S1..S4 of Table 1
SETS = {
    "S1": {"BERT-1.3B": 32},
    "S2": {"BERT-6.7B": 32},
    "S3": {"BERT-1.3B": 10, "BERT-2.7B": 10, "BERT-6.7B": 10,
           "MoE-1.3B": 10, "MoE-2.4B": 10, "MoE-5.3B": 10},
    "S4": {"BERT-104B": 4},
}

DEVICE_BUDGET = 13 * GB  # P:106 footnote
V100_MEMORY = 16 * GB  # P:309 "each GPU has 16GB of memory"
