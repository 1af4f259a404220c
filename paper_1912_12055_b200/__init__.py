"""B200-native (sm_100a) waveform -> spectrogram layers with the capabilities of
nnAudio (arXiv 1912.12055), parity-checked against the `spectro` reference."""

__version__ = "0.1.0"
