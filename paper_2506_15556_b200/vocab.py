"""The fixed-size synthetic vocabulary of the random-init decoder.

The reference's `Vocabulary` (`/root/reference/pkg/src/specstream/text.py:60-122`)
hands out ids in order of first appearance over the run's corpus; a decoder
with a fixed LM head needs a fixed table instead. `SyntheticVocabulary(V)` is a
frozen `specstream.text.Vocabulary` of exactly V ids:

* id 0 is `<eos>` (EOS_ID, text.py:19); ids 1-3 are `.`, `?`, `!` — the
  sentence terminators of text.py:28; every other id `i` is spelled `w<i>`;
* `tokenize` splits with the reference's own `split_words` (text.py:35-57),
  `detokenize` is the reference's (inherited), so `first_sentence`,
  `SentenceTracker` and the event logs see ordinary surfaces.
"""

from __future__ import annotations

from ._specstream import specstream

_text = specstream.text
EOS_ID = _text.EOS_ID
SENTENCE_TERMINATORS = _text.SENTENCE_TERMINATORS


class SyntheticVocabulary(_text.Vocabulary):
    """Frozen `size`-entry table: `<eos>`, `.`, `?`, `!`, then `w4` .. `w<size-1>`."""

    _SPECIAL = (_text.EOS_SURFACE, ".", "?", "!")

    def __init__(self, size: int) -> None:
        if size <= len(self._SPECIAL):
            raise ValueError("synthetic vocabulary needs more than the special ids")
        self._size = size

    def __len__(self) -> int:
        return self._size

    @property
    def frozen(self) -> bool:
        return True

    def freeze(self) -> "SyntheticVocabulary":
        return self

    def surface(self, token_id: int) -> str:
        if not 0 <= token_id < self._size:
            raise _text.VocabularyError(f"token id {token_id} outside vocabulary of size {self._size}")
        if token_id < len(self._SPECIAL):
            return self._SPECIAL[token_id]
        return f"w{token_id}"

    def id_of(self, surface: str) -> int:
        if surface in self._SPECIAL:
            return self._SPECIAL.index(surface)
        if surface[:1] == "w" and surface[1:].isdigit():
            i = int(surface[1:])
            if len(self._SPECIAL) <= i < self._size and surface == f"w{i}":
                return i
        raise _text.VocabularyError(f"unknown surface form {surface!r}")

    # frozen: admitting a surface is a lookup
    add = id_of

    def tokenize(self, text: str) -> list[int]:
        return [self.id_of(w) for w in _text.split_words(text)]

    def word_ids(self) -> range:
        return range(len(self._SPECIAL), self._size)

    def judge_ids(self, text: str) -> list[int]:
        """Token ids for judge text (the consistency-judge template of lm.py:117-131
        is English, which the synthetic table cannot spell): known surfaces keep
        their ids, any other word maps to a word id by 64-bit FNV-1a of its UTF-8
        bytes. One id per `split_words` word, so a pass over it costs what the
        reference's `judge_cost` charges (lm.py:208-213)."""
        out = []
        for w in _text.split_words(text):
            try:
                out.append(self.id_of(w))
            except _text.VocabularyError:
                h = 0xCBF29CE484222325
                for b in w.encode("utf-8"):
                    h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
                out.append(len(self._SPECIAL) + h % (self._size - len(self._SPECIAL)))
        return out


def terminator_mask(vocab) -> bytes:
    """One byte per id, 1 for a sentence terminator (uploaded to the device)."""
    return bytes(1 if vocab.surface(i) in SENTENCE_TERMINATORS else 0 for i in range(len(vocab)))
