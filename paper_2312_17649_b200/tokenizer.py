"""Special token ids (R/tokenizer.py:11-14)."""

CLS_ID = 0
SEP_ID = 1
UNK_ID = 2
NUM_SPECIAL_TOKENS = 3
