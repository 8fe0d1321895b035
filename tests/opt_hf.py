"""Map the flat ranker parameter dict onto transformers' OPTModel (the third-party
implementation that pins oracle/opt_ranker.py; transformers is in the image)."""

import torch


def hf_model(cfg, params):
    from transformers import OPTConfig, OPTModel
    hc = OPTConfig(vocab_size=cfg.vocab, hidden_size=cfg.d_model, num_hidden_layers=cfg.n_layers,
                   ffn_dim=cfg.d_ffn, num_attention_heads=cfg.n_heads, max_position_embeddings=cfg.max_pos,
                   word_embed_proj_dim=cfg.d_model, do_layer_norm_before=True, dropout=0.0,
                   attention_dropout=0.0, activation_dropout=0.0, layerdrop=0.0,
                   activation_function="relu" if cfg.activation == 0 else "gelu_new", enable_bias=True)
    m = OPTModel(hc).eval()
    d = cfg.d_model
    sd = {"decoder.embed_tokens.weight": params["tok_emb"], "decoder.embed_positions.weight": params["pos_emb"],
          "decoder.final_layer_norm.weight": params["lnf_w"], "decoder.final_layer_norm.bias": params["lnf_b"]}
    for i in range(cfg.n_layers):
        p = lambda k: params[f"layers.{i}.{k}"]  # noqa: E731
        pre = f"decoder.layers.{i}."
        for j, nm in enumerate("qkv"):
            sd[pre + f"self_attn.{nm}_proj.weight"] = p("qkv_w")[j * d:(j + 1) * d]
            sd[pre + f"self_attn.{nm}_proj.bias"] = p("qkv_b")[j * d:(j + 1) * d]
        sd[pre + "self_attn.out_proj.weight"] = p("out_w")
        sd[pre + "self_attn.out_proj.bias"] = p("out_b")
        sd[pre + "self_attn_layer_norm.weight"] = p("ln1_w")
        sd[pre + "self_attn_layer_norm.bias"] = p("ln1_b")
        sd[pre + "final_layer_norm.weight"] = p("ln2_w")
        sd[pre + "final_layer_norm.bias"] = p("ln2_b")
        sd[pre + "fc1.weight"], sd[pre + "fc1.bias"] = p("fc1_w"), p("fc1_b")
        sd[pre + "fc2.weight"], sd[pre + "fc2.bias"] = p("fc2_w"), p("fc2_b")
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected, unexpected
    assert all("project" in k for k in missing), missing
    return m


@torch.no_grad()
def hf_scores(cfg, params, ids, last_pos=None):
    m = hf_model(cfg, params)
    ids = torch.as_tensor(ids).long()
    h = m(input_ids=ids).last_hidden_state  # after decoder.final_layer_norm
    B, S = ids.shape
    lp = torch.full((B,), S - 1) if last_pos is None else torch.as_tensor(last_pos).long()
    return h[torch.arange(B), lp] @ params["head_w"] + params["head_b"][0]
