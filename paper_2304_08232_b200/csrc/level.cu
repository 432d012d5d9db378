// level.cu — multigrid levels (problem.hpp:220-319), the coloured Gauss-Seidel smoother
// (smoother.hpp) and the V-cycle (multigrid.hpp) on top of the kernels.
#include <algorithm>
#include <limits>

#include "common.hpp"
#include "dist.hpp"
#include "kernels.cuh"

slab_level_s::~slab_level_s() {
	colorA.release();
	tile.release();
	if( d_rows ) {
		cudaFree( d_rows );
	}
	if( vcycle_exec ) {
		cudaGraphExecDestroy( vcycle_exec );
	}
	slabgpu::halo_plan_destroy( plan );
}

namespace slabgpu {

	// ---------------------------------------------------------------- LevelStats timing

	namespace {
		cudaEvent_t event_get( slab_ctx_s * ctx ) {
			if( !ctx->event_pool.empty() ) {
				cudaEvent_t e = ctx->event_pool.back();
				ctx->event_pool.pop_back();
				return e;
			}
			cudaEvent_t e = nullptr;
			SLAB_CUDA( cudaEventCreate( &e ) );
			return e;
		}

		// records the interval [construction, destruction) on the context's stream when profiling is on
		struct Span {
			slab_ctx_s * ctx;
			uint64_t * target;
			int sign;
			cudaEvent_t begin = nullptr;
			Span( slab_ctx_s * c, uint64_t * t, int s = 1 ) : ctx( c ), target( t ), sign( s ) {
				if( ctx->profiling ) {
					begin = event_get( ctx );
					SLAB_CUDA( cudaEventRecord( begin, ctx->stream ) );
				}
			}
			~Span() {
				if( begin != nullptr ) {
					cudaEvent_t end = event_get( ctx );
					cudaEventRecord( end, ctx->stream );
					ctx->spans.push_back( { begin, end, target, sign } );
				}
			}
		};
	} // namespace

	void spans_resolve( slab_ctx_s * ctx ) {
		if( ctx->spans.empty() ) {
			return;
		}
		SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) );
		for( const TimedSpan & span : ctx->spans ) {
			float ms = 0.0f;
			if( cudaEventElapsedTime( &ms, span.begin, span.end ) == cudaSuccess ) {
				const uint64_t ns = static_cast< uint64_t >( static_cast< double >( ms ) * 1e6 );
				if( span.sign > 0 ) {
					*span.target += ns;
				} else {
					*span.target -= ns < *span.target ? ns : *span.target;
				}
			}
			ctx->event_pool.push_back( span.begin );
			ctx->event_pool.push_back( span.end );
		}
		ctx->spans.clear();
	}

	void spans_discard( slab_ctx_s * ctx ) {
		for( const TimedSpan & span : ctx->spans ) {
			ctx->event_pool.push_back( span.begin );
			ctx->event_pool.push_back( span.end );
		}
		ctx->spans.clear();
	}

	namespace {

		int64_t round_up( int64_t v, int64_t m ) {
			return ( v + m - 1 ) / m * m;
		}

		void alloc_scratch( slab_level_s * L, uint64_t n_coarse ) {
			L->f.reset( vec_new( L->ctx, L->n, 0.0 ) );
			if( n_coarse > 0 ) {
				L->r_c.reset( vec_new( L->ctx, n_coarse, 0.0 ) );
				L->z_c.reset( vec_new( L->ctx, n_coarse, 0.0 ) );
			}
		}

		// One stencil level, generated on the device. The colouring is the closed form of what
		// greedy_color (coloring.hpp:114-158) finds on every 27-point grid: colour k is the parity
		// class ix%2 + 2*(iy%2) + 4*(iz%2), members ascending (tests pin this against the oracle's
		// greedy colouring, even and odd dimensions).
		slab_level_s * stencil_level( slab_ctx_s * ctx, uint64_t nx, uint64_t ny, uint64_t nz, bool with_restriction ) {
			std::unique_ptr< slab_level_s > L( new slab_level_s );
			L->ctx = ctx;
			L->dims[ 0 ] = nx;
			L->dims[ 1 ] = ny;
			L->dims[ 2 ] = nz;
			L->is_stencil = true;
			// the box this rank owns (the whole grid on a single-process context); colours are the
			// parity classes of the GLOBAL coordinates, so they agree with the single-process
			// colouring even where a rank's offset is odd
			const Decomp D = level_decomp( ctx, nx, ny, nz );
			L->decomp = D;
			L->A.reset( mat_stencil27_box( ctx, D ) );
			L->n = L->A->nrows;
			L->nnz = L->A->nnz;
			if( ctx->dist != nullptr ) {
				L->plan = halo_plan_create( ctx, D );
				L->A->plan = L->plan;
			}
			L->num_colors = 8;
			L->color_pos.assign( 9, 0 );
			L->color_size.assign( 8, 0 );
			L->color_nnz.assign( 8, 0 );
			for( int k = 0; k < 8; ++k ) {
				const int c[ 3 ] = { k & 1, ( k >> 1 ) & 1, ( k >> 2 ) & 1 };
				uint64_t size = 1, cnnz = 1;
				for( int a = 0; a < 3; ++a ) {
					size *= static_cast< uint64_t >( count_parity( D.o[ a ], D.l[ a ], c[ a ] ) );
					uint64_t spans = 0;
					for( int t = first_parity( D.o[ a ], c[ a ] ); t < D.o[ a ] + D.l[ a ]; t += 2 ) {
						spans += static_cast< uint64_t >( span_1d( t, D.g[ a ] ) );
					}
					cnnz *= spans;
				}
				L->color_size[ k ] = size;
				L->color_nnz[ k ] = cnnz;
				L->color_pos[ k + 1 ] = L->color_pos[ k ] + round_up( static_cast< int64_t >( size ), kSlice );
			}
			const int64_t npos = L->color_pos[ 8 ];
			if( L->plan != nullptr && D.n_ghost > 0 ) {
				// boundary rows of every colour, as positions of the colour-major order
				std::vector< std::vector< int32_t > > boundary( 8 );
				for( int c = 0; c < 8; ++c ) {
					const int cc[ 3 ] = { c & 1, ( c >> 1 ) & 1, ( c >> 2 ) & 1 };
					const int sx = count_parity( D.o[ 0 ], D.l[ 0 ], cc[ 0 ] ), sy = count_parity( D.o[ 1 ], D.l[ 1 ], cc[ 1 ] );
					std::vector< int32_t > positions;
					for( int dir = 0; dir < 27; ++dir ) {
						if( dir == 13 || D.ghost_count[ dir ][ 0 ] + D.ghost_count[ dir ][ 1 ] + D.ghost_count[ dir ][ 2 ]
								+ D.ghost_count[ dir ][ 3 ] + D.ghost_count[ dir ][ 4 ] + D.ghost_count[ dir ][ 5 ] + D.ghost_count[ dir ][ 6 ]
								+ D.ghost_count[ dir ][ 7 ] == 0 ) {
							continue; // no neighbour in that direction
						}
						std::vector< int32_t > list;
						send_list( D, dir, c, list );
						for( const int32_t idx : list ) {
							const int ix = idx % D.l[ 0 ], iy = ( idx / D.l[ 0 ] ) % D.l[ 1 ], iz = idx / ( D.l[ 0 ] * D.l[ 1 ] );
							const int qx = ( D.o[ 0 ] + ix - first_parity( D.o[ 0 ], cc[ 0 ] ) ) >> 1;
							const int qy = ( D.o[ 1 ] + iy - first_parity( D.o[ 1 ], cc[ 1 ] ) ) >> 1;
							const int qz = ( D.o[ 2 ] + iz - first_parity( D.o[ 2 ], cc[ 2 ] ) ) >> 1;
							positions.push_back( static_cast< int32_t >( L->color_pos[ c ] + qx + static_cast< int64_t >( sx ) * ( qy + static_cast< int64_t >( sy ) * qz ) ) );
						}
					}
					std::sort( positions.begin(), positions.end() );
					positions.erase( std::unique( positions.begin(), positions.end() ), positions.end() );
					boundary[ c ] = std::move( positions );
				}
				halo_plan_set_boundary( ctx, L->plan, boundary, npos );
			}
			SLAB_CUDA( cudaMalloc( &L->d_rows, std::max< int64_t >( npos, 1 ) * sizeof( int32_t ) ) );
			for( int k = 0; k < 8; ++k ) {
				kern::color_rows( ctx->stream, D, k, L->color_pos[ k ], static_cast< int64_t >( L->color_size[ k ] ),
					L->color_pos[ k + 1 ] - L->color_pos[ k ], L->d_rows );
			}
			L->colorA = sell_stencil27( ctx, D, L->d_rows, npos );
			sell_pack( ctx, L->colorA, L->d_rows, static_cast< int64_t >( L->n ) ); // columns >= n are ghost slots
			// rows as masks over the 27 offsets, for the shared-memory-staged colour-pair kernel (tile.cu): single
			// process only (no ghost columns), and only if the row list is the parity lattice that kernel assumes
			if( ctx->dist == nullptr && D.n_ghost == 0 && L->colorA.packed.usable() && ( D.l[ 0 ] % 2 ) == 0
				&& box_tile_lattice_ok( ctx, L->d_rows, L->color_pos, D ) ) {
				box_tile_build( ctx, L->colorA, L->d_rows, D, L->tile );
				// (whether a level of this size takes the plane phases is decided per call, planes_usable: here only whether it could)
				if( L->tile.usable() && kern::gs_planes_usable( L->tile, std::numeric_limits< int64_t >::max(), ctx->sm_count ) ) {
					L->planes_ok = true;
					L->zs.reset( vec_new( ctx, L->n, 0.0 ) );
					kern::gs_planes_prepare();
				}
			}
			L->a_diag.reset( vec_new( ctx, L->n, 26.0 ) ); // extract_diagonal of the stencil: 26.0 everywhere
			uint64_t n_coarse = 0;
			if( with_restriction ) {
				L->R.reset( mat_restriction( ctx, nx, ny, nz ) );
				n_coarse = L->R->nrows;
			}
			alloc_scratch( L.get(), n_coarse );
			if( L->planes_ok ) {
				// the level measures the tile shapes its cost models propose for the three phases of a sweep (plane.cu)
				std::unique_ptr< slab_vec_s > tmp( vec_new( ctx, L->n, 0.0 ) );
				kern::gs_planes_tune( ctx->stream, ctx->sm_count, L->tile, tmp->d, L->zs->d, L->f->d );
				kern::fill( ctx->stream, L->zs->d, L->n, 0.0 );
				kern::fill( ctx->stream, L->f->d, L->n, 0.0 );
				SLAB_CUDA( cudaStreamSynchronize( ctx->stream ) ); // tmp goes away
			}
			return L.release();
		}

	} // namespace

	// problem.hpp:284-319
	slab_level_s * hierarchy_create( slab_ctx_s * ctx, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t levels ) {
		if( nx < 2 || ny < 2 || nz < 2 ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "grid dimensions must all be at least 2, got " + std::to_string( nx ) + "x"
				+ std::to_string( ny ) + "x" + std::to_string( nz ) );
		}
		{ // the row count must fit 32-bit column indices; checked without letting the product wrap
			const uint64_t limit = uint64_t( 1 ) << 31;
			if( nx >= limit || ny >= limit || nz >= limit || nx > ( limit - 1 ) / ny || nx * ny > ( limit - 1 ) / nz ) {
				fail( SLAB_ERR_INVALID_ARGUMENT, "grid too large for 32-bit column indices on one device" );
			}
		}
		if( levels < 1 ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "build_hierarchy: need at least one level" );
		}
		if( levels > 40 ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "build_hierarchy: too many levels" );
		}
		const uint64_t divider = uint64_t( 1 ) << ( levels - 1 );
		const uint64_t d[ 3 ] = { nx, ny, nz };
		const char * names[ 3 ] = { "nx", "ny", "nz" };
		for( int a = 0; a < 3; ++a ) {
			if( d[ a ] % divider != 0 ) {
				fail( SLAB_ERR_INVALID_ARGUMENT, std::string( "build_hierarchy: dimension " ) + names[ a ] + " = "
					+ std::to_string( d[ a ] ) + " is not divisible by 2^(levels-1) = " + std::to_string( divider ) );
			}
			if( d[ a ] / divider < 2 ) {
				fail( SLAB_ERR_INVALID_ARGUMENT, std::string( "build_hierarchy: dimension " ) + names[ a ] + " = "
					+ std::to_string( d[ a ] ) + " becomes smaller than 2 after " + std::to_string( levels - 1 ) + " halvings" );
			}
		}
		std::unique_ptr< slab_level_s > head;
		slab_level_s * tail = nullptr;
		uint64_t lx = nx, ly = ny, lz = nz;
		for( uint64_t k = 0; k < levels; ++k ) {
			std::unique_ptr< slab_level_s > L( stencil_level( ctx, lx, ly, lz, k + 1 < levels ) );
			slab_level_s * raw = L.get();
			if( tail == nullptr ) {
				head = std::move( L );
			} else {
				tail->coarser = std::move( L );
			}
			tail = raw;
			lx /= 2;
			ly /= 2;
			lz /= 2;
		}
		return head.release();
	}

	// ProblemLevel(SparseMatrix) problem.hpp:253 for an arbitrary square system: extract_diagonal
	// (problem.hpp:143-166) over the host CSR the caller handed in, greedy_color (coloring.hpp:114-158) on the
	// device (coloring.cu), the rows of a colour in ascending order (coloring.hpp:148-151).
	slab_level_s * level_from_csr( slab_ctx_s * ctx, uint64_t n, const uint64_t * ro, const uint64_t * co,
		const double * va ) {
		std::unique_ptr< slab_level_s > L( new slab_level_s );
		L->ctx = ctx;
		L->dims[ 0 ] = n;
		L->dims[ 1 ] = 1;
		L->dims[ 2 ] = 1;
		L->A.reset( mat_from_csr( ctx, n, n, ro, co, va, true ) );
		L->n = n;
		L->nnz = L->A->nnz;

		std::vector< double > diag( n );
		for( uint64_t i = 0; i < n; ++i ) {
			const uint64_t * first = co + ro[ i ];
			const uint64_t * last = co + ro[ i + 1 ];
			const uint64_t * hit = std::lower_bound( first, last, i );
			if( hit == last || *hit != i || va[ hit - co ] == 0.0 ) {
				fail( SLAB_ERR_INVALID_ARGUMENT, "extract_diagonal: row " + std::to_string( i ) + " has no usable diagonal entry" );
			}
			diag[ i ] = va[ hit - co ];
		}

		// greedy_color on the device (coloring.cu): colour(i) = smallest colour no lower-index neighbour of
		// pattern(A) united with pattern(A^T) has — the sequential result, evaluated as a wavefront
		std::vector< int32_t > color;
		uint64_t num_colors = 0;
		greedy_color_device( ctx, n, ro, co, color, num_colors );

		L->num_colors = num_colors;
		L->color_size.assign( num_colors, 0 );
		L->color_nnz.assign( num_colors, 0 );
		for( uint64_t i = 0; i < n; ++i ) {
			++L->color_size[ color[ i ] ];
			L->color_nnz[ color[ i ] ] += ro[ i + 1 ] - ro[ i ];
		}
		L->color_pos.assign( num_colors + 1, 0 );
		for( uint64_t k = 0; k < num_colors; ++k ) {
			L->color_pos[ k + 1 ] = L->color_pos[ k ] + round_up( static_cast< int64_t >( L->color_size[ k ] ), kSlice );
		}
		std::vector< int64_t > rows( L->color_pos[ num_colors ], -1 );
		std::vector< int64_t > fill( L->color_pos.begin(), L->color_pos.end() - 1 );
		for( uint64_t i = 0; i < n; ++i ) {
			rows[ fill[ color[ i ] ]++ ] = static_cast< int64_t >( i ); // ascending i keeps members sorted
		}
		L->colorA = sell_from_csr_rows( ctx, rows, ro, co, va );
		std::vector< int32_t > rows32( rows.begin(), rows.end() );
		SLAB_CUDA( cudaMalloc( &L->d_rows, std::max< size_t >( rows32.size(), 1 ) * sizeof( int32_t ) ) );
		upload_sync( ctx->stream, L->d_rows, rows32.data(), rows32.size() * sizeof( int32_t ) );
		sell_pack( ctx, L->colorA, L->d_rows );
		L->a_diag.reset( vec_new( ctx, n, 0.0 ) );
		upload_sync( ctx->stream, L->a_diag->d, diag.data(), n * sizeof( double ) );
		alloc_scratch( L.get(), 0 );
		return L.release();
	}

	// ---------------------------------------------------------------- smoother.hpp

	namespace {
		void check_smoother_args( slab_level_s * L, slab_vec_s * z, slab_vec_s * r ) { // smoother.hpp:54-58
			if( z->n != L->n || r->n != L->n ) {
				fail( SLAB_ERR_DIMENSION_MISMATCH, "smoother: vector lengths differ from the level size" );
			}
		}

		// One colour step. Invariant on distributed levels: the ghost copies of z are current on
		// entry; the step then sends the just-updated boundary values of colour k to the neighbours
		// (only that colour moved), which restores the invariant for the next step.
		void color_step_enqueue( slab_level_s * L, uint64_t k, slab_vec_s * z, slab_vec_s * r, int flags = 0 ) {
			slab_ctx_s * ctx = L->ctx;
			const double * src = ( flags & 1 ) ? L->z_c->d : nullptr;
			double * out = ( flags & 2 ) ? L->r_c->d : nullptr;
			double * zero = ( flags & 2 ) ? L->z_c->d : nullptr;
			const size_t window = static_cast< size_t >( z->n_alloc ) * sizeof( double );
			const int64_t count = static_cast< int64_t >( L->color_size[ k ] );
			if( !halo_overlap_active( ctx, L->plan ) ) {
				kern::gs_color_step( ctx->stream, L->colorA, L->d_rows,
					L->color_pos[ k ], count, z->d, r->d, flags, src, out, zero, window );
				halo_exchange( L, z, static_cast< int >( k ) );
				return;
			}
			// Distributed level: (1) the boundary rows of the colour, (2) their halo messages on the
			// communication stream, (3) the interior rows on the main stream meanwhile, (4) join. Interior rows
			// have no ghost neighbours and nobody reads the colour's ghost slots during this step, so the
			// two streams touch disjoint data. Same arithmetic per row as the single launch.
			int64_t nb = 0;
			const int32_t * bpos = halo_boundary_positions( L->plan, static_cast< int >( k ), &nb );
			if( nb > 0 ) {
				kern::gs_color_step( ctx->stream, L->colorA, L->d_rows,
					L->color_pos[ k ], nb, z->d, r->d, flags, src, out, zero, 0, bpos, nullptr );
			}
			const bool comm = halo_has_comm( ctx );
			if( comm ) {
				halo_fork( ctx );
				halo_exchange_plan( ctx, L->plan, z, static_cast< int >( k ), halo_comm_stream( ctx ) );
			}
			kern::gs_color_step( ctx->stream, L->colorA, L->d_rows,
				L->color_pos[ k ], count, z->d, r->d, flags, src, out, zero, window, nullptr, halo_boundary_flags( L->plan ) );
			if( comm ) {
				halo_join( ctx );
			}
		}

		// the colour-pair kernel of tile.cu serves this level? (stencil level on one process, masks built and checked)
		bool tile_pairs_usable( const slab_level_s * L ) {
			return L->is_stencil && L->plan == nullptr && L->num_colors == 8
				&& kern::gs_pair_tile_usable( L->tile, static_cast< int64_t >( L->color_size[ 0 ] + L->color_size[ 1 ] ) );
		}

		void tile_pair_enqueue( slab_level_s * L, int pair, int mode, slab_vec_s * z, slab_vec_s * r, int flags ) {
			kern::gs_pair_tile( L->ctx->stream, L->ctx->sm_count, L->tile, L->color_pos, pair, mode, z->d, r->d, flags,
				( flags & 1 ) ? L->z_c->d : nullptr, ( flags & 2 ) ? L->r_c->d : nullptr, ( flags & 2 ) ? L->z_c->d : nullptr );
		}

		// the three-launch plane phases of plane.cu serve this level? (regular stencil box on one process)
		bool planes_usable( const slab_level_s * L ) {
			return L->planes_ok && g_use_planes && L->plan == nullptr && static_cast< int64_t >( L->n ) >= g_plane_min_rows;
		}

		void plane_phase_enqueue( slab_level_s * L, int kind, int pass, const double * own_in, const double * nb_in, double * own_out,
			double * pass_out, slab_vec_s * r, int flags ) {
			// flags bit 4: r'z partials, phase B's blocks first, phase C's behind them (cg.cu folds them in that order)
			double * dot_partials = nullptr;
			if( flags & 16 ) {
				dot_partials = L->ctx->d_partials + ( kind == 2 ? kern::gs_planes_blocks( L->tile, 1, L->ctx->sm_count ) : 0 );
			}
			kern::gs_planes( L->ctx->stream, L->ctx->sm_count, L->tile, kind, pass, own_in, nb_in, own_out, pass_out, r->d, flags,
				( flags & 1 ) ? L->z_c->d : nullptr, ( flags & 2 ) ? L->r_c->d : nullptr, ( flags & 2 ) ? L->z_c->d : nullptr, dot_partials );
		}

		void forward_enqueue( slab_level_s * L, slab_vec_s * z, slab_vec_s * r ) { // smoother.hpp:80-82
			if( planes_usable( L ) ) {
				double * const zs = L->zs->d;
				plane_phase_enqueue( L, 0, 1, z->d, z->d, zs, zs, r, 0 );     // colours 0..3: z -> zs, odd planes copied along
				plane_phase_enqueue( L, 3, 2 | 4, zs, zs, z->d, z->d, r, 0 ); // colours 4..7: zs -> z, even planes copied along
				return;
			}
			if( tile_pairs_usable( L ) ) {
				for( int p = 0; p < 4; ++p ) {
					tile_pair_enqueue( L, p, 0, z, r, 0 );
				}
				return;
			}
			for( uint64_t k = 0; k < L->num_colors; ++k ) {
				color_step_enqueue( L, k, z, r );
			}
		}

		void backward_enqueue( slab_level_s * L, slab_vec_s * z, slab_vec_s * r ) { // smoother.hpp:95-97
			if( planes_usable( L ) ) {
				double * const zs = L->zs->d;
				plane_phase_enqueue( L, 4, 2 | 4, z->d, z->d, zs, zs, r, 0 ); // colours 7..4: z -> zs, even planes copied along
				plane_phase_enqueue( L, 2, 1, zs, zs, z->d, z->d, r, 0 );     // colours 3..0: zs -> z, odd planes copied along
				return;
			}
			if( tile_pairs_usable( L ) ) {
				for( int p = 3; p >= 0; --p ) {
					tile_pair_enqueue( L, p, 1, z, r, 0 );
				}
				return;
			}
			for( uint64_t k = L->num_colors; k > 0; --k ) {
				color_step_enqueue( L, k - 1, z, r );
			}
		}

		// One forward + one backward sweep (smoother.hpp:108-111). The last colour of the forward sweep is the
		// first of the backward sweep and nothing but its own entries changes in between, so that step is ONE
		// launch whose threads apply the update twice (flags bit 2) — one launch and one pass over the colour's
		// matrix rows less per symmetric sweep, same arithmetic in the same order. On a decomposed level the
		// halo message of that colour goes out once, after the second update: the rows of a colour never read
		// the colour's own ghost copies, so nobody misses the intermediate values.
		// first_flags / last_flags ride on the first forward and the last backward step (grid transfers).
		void sweep_pair_enqueue( slab_level_s * L, slab_vec_s * z, slab_vec_s * r, int first_flags = 0, int last_flags = 0 ) {
			const uint64_t nc = L->num_colors;
			if( planes_usable( L ) ) {
				// plane.cu: even planes (colours 0-3), odd planes (4-7, 7-4), even planes (3-0); every phase out of place
				double * const zs = L->zs->d;
				plane_phase_enqueue( L, 0, 1, z->d, z->d, zs, zs, r, first_flags & ( 1 | 8 ) ); // z -> zs, odd planes copied along
				plane_phase_enqueue( L, 1, 0, zs, zs, z->d, nullptr, r, last_flags & 16 );    // odd planes: zs -> z
				plane_phase_enqueue( L, 2, 0, zs, z->d, z->d, nullptr, r, last_flags & ( 2 | 16 ) ); // even planes: zs (+ odd planes of z) -> z
				return;
			}
			// small level on one process: the whole pair of sweeps in one launch (sweep_cluster.cu), same steps
			if( L->ctx->fused_transfers && L->plan == nullptr && nc >= 1
				&& kern::gs_sweep_cluster_usable( L->colorA, L->color_pos, L->color_size, L->n ) ) {
				const int flags = first_flags | last_flags;
				kern::gs_sweep_cluster( L->ctx->stream, L->colorA, L->d_rows, L->color_pos, L->color_size, L->n, z->d, r->d,
					first_flags, last_flags, ( flags & 1 ) ? L->z_c->d : nullptr, ( flags & 2 ) ? L->r_c->d : nullptr,
					( flags & 2 ) ? L->z_c->d : nullptr );
				return;
			}
			if( tile_pairs_usable( L ) ) {
				// colour pairs (2p, 2p+1) as single launches (tile.cu); 7 launches per symmetric sweep with the turnaround
				const bool turn = L->ctx->fused_transfers != 0;
				for( int p = 0; p < 3; ++p ) {
					tile_pair_enqueue( L, p, 0, z, r, p == 0 ? first_flags : 0 );
				}
				if( turn ) {
					tile_pair_enqueue( L, 3, 2, z, r, 0 );
				} else {
					tile_pair_enqueue( L, 3, 0, z, r, 0 );
					tile_pair_enqueue( L, 3, 1, z, r, 0 );
				}
				for( int p = 2; p >= 0; --p ) {
					tile_pair_enqueue( L, p, 1, z, r, p == 0 ? last_flags : 0 );
				}
				return;
			}
			const bool turnaround = L->ctx->fused_transfers && nc >= 2
				&& kern::gs_color_step_can_fuse_residual( L->colorA, static_cast< int64_t >( L->color_size[ nc - 1 ] ) );
			for( uint64_t k = 0; k < nc; ++k ) {
				const int flags = ( k == 0 ? first_flags : 0 ) | ( turnaround && k + 1 == nc ? 4 : 0 );
				color_step_enqueue( L, k, z, r, flags );
			}
			for( uint64_t k = turnaround ? nc - 1 : nc; k > 0; --k ) {
				color_step_enqueue( L, k - 1, z, r, k == 1 ? last_flags : 0 );
			}
		}

		// zero_guess: z is known to be zero on entry; levels that run the plane phases then do not read it in the first
		// phase of the first sweep (first_flags bit 3), every other path ignores the hint
		// fuse_rz: the last sweep also leaves the partials of r'z behind (last_flags bit 4; plane phases only)
		void symmetric_enqueue( slab_level_s * L, slab_vec_s * z, slab_vec_s * r, uint64_t sweeps, bool zero_guess = false, bool fuse_rz = false ) { // smoother.hpp:108-111
			for( uint64_t sweep = 0; sweep < sweeps; ++sweep ) {
				sweep_pair_enqueue( L, z, r, sweep == 0 && zero_guess && planes_usable( L ) ? 8 : 0,
					sweep + 1 == sweeps && fuse_rz && planes_usable( L ) ? 16 : 0 );
			}
		}
	} // namespace

	void rbgs_color_step( slab_level_s * L, uint64_t k, slab_vec_s * z, slab_vec_s * r ) {
		check_smoother_args( L, z, r );
		if( k >= L->num_colors ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "rbgs_color_step: colour index out of range" );
		}
		halo_exchange( L, z, -1 ); // z is the caller's: its ghost copies may be stale
		color_step_enqueue( L, k, z, r );
		L->stats.nnz_visited += L->color_nnz[ k ]; // smoother.hpp:71
	}

	// the same step applied twice in a row by one launch (the turnaround of a symmetric sweep); falls back to two
	// steps where the kernel shape cannot repeat
	void rbgs_color_step_twice( slab_level_s * L, uint64_t k, slab_vec_s * z, slab_vec_s * r ) {
		check_smoother_args( L, z, r );
		if( k >= L->num_colors ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "rbgs_color_step_twice: colour index out of range" );
		}
		halo_exchange( L, z, -1 );
		if( kern::gs_color_step_can_fuse_residual( L->colorA, static_cast< int64_t >( L->color_size[ k ] ) ) ) {
			color_step_enqueue( L, k, z, r, 4 );
		} else {
			color_step_enqueue( L, k, z, r );
			color_step_enqueue( L, k, z, r );
		}
		L->stats.nnz_visited += 2 * L->color_nnz[ k ];
	}

	void rbgs_forward( slab_level_s * L, slab_vec_s * z, slab_vec_s * r ) {
		check_smoother_args( L, z, r );
		halo_exchange( L, z, -1 );
		{
			Span timed( L->ctx, &L->stats.smoother_ns ); // smoother.hpp:79,83
			forward_enqueue( L, z, r );
		}
		L->stats.nnz_visited += L->nnz;
	}

	void rbgs_backward( slab_level_s * L, slab_vec_s * z, slab_vec_s * r ) {
		check_smoother_args( L, z, r );
		halo_exchange( L, z, -1 );
		{
			Span timed( L->ctx, &L->stats.smoother_ns ); // smoother.hpp:94,98
			backward_enqueue( L, z, r );
		}
		L->stats.nnz_visited += L->nnz;
	}

	void rbgs_symmetric( slab_level_s * L, slab_vec_s * z, slab_vec_s * r, uint64_t sweeps ) {
		if( sweeps < 1 ) { // smoother.hpp:105-107
			fail( SLAB_ERR_INVALID_ARGUMENT, "SmootherConfig: sweeps must be at least 1" );
		}
		check_smoother_args( L, z, r );
		halo_exchange( L, z, -1 );
		{
			Span timed( L->ctx, &L->stats.smoother_ns );
			symmetric_enqueue( L, z, r, sweeps );
		}
		L->stats.nnz_visited += 2 * sweeps * L->nnz;
	}

	// ---------------------------------------------------------------- multigrid.hpp

	void restrict_vector( slab_level_s * L, slab_vec_s * v_fine, slab_vec_s * out ) { // multigrid.hpp:46-54
		if( !L->R ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "restrict_vector: the coarsest level has no restriction operator" );
		}
		{
			Span timed( L->ctx, &L->stats.transfer_ns ); // multigrid.hpp:50-52
			op_mxv( out, nullptr, L->R.get(), v_fine, SLAB_DESC_NONE );
		}
		L->stats.nnz_visited += L->R->nnz;
	}

	void refine_and_add( slab_level_s * L, slab_vec_s * z, slab_vec_s * z_c ) { // multigrid.hpp:71-81
		if( !L->R ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "refine_and_add: the coarsest level has no restriction operator" );
		}
		if( z_c->n != L->R->nrows || z->n != L->n ) {
			fail( SLAB_ERR_DIMENSION_MISMATCH, "mxv: operand sizes do not match the matrix" );
		}
		{
			Span timed( L->ctx, &L->stats.transfer_ns ); // multigrid.hpp:75-78
			if( L->ctx->fused_transfers ) {
				// injected rows are the colour-0 block: position p <-> coarse index p
				kern::prolong_add( L->ctx->stream, L->d_rows, static_cast< int64_t >( z_c->n ), z->d, z_c->d );
			} else {
				op_mxv( L->f.get(), nullptr, L->R.get(), z_c, SLAB_DESC_TRANSPOSE );
				op_waxpby( z, 1.0, z, 1.0, L->f.get() );
			}
		}
		L->stats.nnz_visited += L->R->nnz;
	}

	namespace {
		void vcycle_stats( slab_level_s * L, uint64_t sweeps ) {
			if( !L->coarser ) {
				L->stats.nnz_visited += 2 * sweeps * L->nnz;
				return;
			}
			// two symmetric smooths, the residual pass, restriction and refinement
			L->stats.nnz_visited += 4 * sweeps * L->nnz + L->nnz + 2 * L->R->nnz;
			vcycle_stats( L->coarser.get(), sweeps );
		}
	} // namespace

	void mg_vcycle_prepare( slab_level_s * L, slab_vec_s * z, slab_vec_s * r, uint64_t sweeps ) {
		slab_ctx_s * ctx = L->ctx;
		if( !ctx->fused_transfers ) {
			for( slab_level_s * at = L; at && at->R; at = at->coarser.get() ) {
				mat_transposed( at->R.get() ); // built lazily; allocation is illegal during capture
			}
		}
		(void) z;
		(void) r;
		(void) sweeps;
	}

	// multigrid.hpp:87-116, enqueue only (no checks, no host synchronisation): safe under stream capture
	bool mg_vcycle_accepts_zero_guess( const slab_level_s * L ) {
		const slab_ctx_s * ctx = L->ctx;
		return !ctx->profiling && planes_usable( L ) && ( !L->coarser || ( ctx->fused_transfers && L->is_stencil ) );
	}

	// zero_guess: the caller knows z to be zero (cg.hpp:111; the coarse guesses of multigrid.hpp:104)
	uint64_t mg_vcycle_rz_partials( const slab_level_s * L ) {
		return kern::gs_planes_blocks( L->tile, 1, L->ctx->sm_count ) + kern::gs_planes_blocks( L->tile, 2, L->ctx->sm_count );
	}

	// fuse_rz: the last phases of the last sweep leave the partials of r'z in the context's reduction scratch
	// (only where mg_vcycle_accepts_zero_guess holds; cg.cu folds them)
	void mg_vcycle_enqueue( slab_level_s * L, slab_vec_s * z, slab_vec_s * r, uint64_t sweeps, bool count_stats, bool zero_guess, bool fuse_rz ) {
		slab_ctx_s * ctx = L->ctx;
		if( ctx->profiling ) {
			// the reference's instrumentation (multigrid.hpp:92-114, smoother.hpp:79-98): per-level V-cycle
			// time with the coarser levels subtracted, smoother and transfer time inside it. Launch by
			// launch, transfers as their own kernels so that they can be attributed.
			Span whole( ctx, &L->stats.mg_ns );
			{
				Span smooth( ctx, &L->stats.smoother_ns );
				symmetric_enqueue( L, z, r, sweeps );
			}
			if( L->coarser ) {
				if( ctx->fused_transfers && L->is_stencil ) {
					Span transfer( ctx, &L->stats.transfer_ns ); // residual + restriction in one kernel
					kern::residual_restrict( ctx->stream, L->colorA, L->d_rows,
						static_cast< int64_t >( L->r_c->n ), z->d, r->d, L->r_c->d, nullptr );
				} else {
					op_mxv( L->f.get(), nullptr, L->A.get(), z, SLAB_DESC_NONE );
					op_waxpby( L->f.get(), 1.0, r, -1.0, L->f.get() );
					Span transfer( ctx, &L->stats.transfer_ns );
					op_mxv( L->r_c.get(), nullptr, L->R.get(), L->f.get(), SLAB_DESC_NONE );
				}
				op_set_all( L->z_c.get(), 0.0 );
				{
					Span child( ctx, &L->stats.mg_ns, -1 ); // per-level time excludes the coarser levels
					mg_vcycle_enqueue( L->coarser.get(), L->z_c.get(), L->r_c.get(), sweeps, count_stats );
				}
				{
					Span transfer( ctx, &L->stats.transfer_ns );
					if( ctx->fused_transfers && L->is_stencil ) {
						kern::prolong_add( ctx->stream, L->d_rows, static_cast< int64_t >( L->z_c->n ), z->d, L->z_c->d );
					} else {
						op_mxv( L->f.get(), nullptr, L->R.get(), L->z_c.get(), SLAB_DESC_TRANSPOSE );
						op_waxpby( z, 1.0, z, 1.0, L->f.get() );
					}
				}
				if( L->plan != nullptr ) {
					halo_exchange( L, z, 0 ); // the separate prolongation changed colour-0 boundary values
				}
				Span smooth( ctx, &L->stats.smoother_ns );
				symmetric_enqueue( L, z, r, sweeps );
			}
			if( count_stats ) {
				L->stats.nnz_visited += L->coarser ? 4 * sweeps * L->nnz + L->nnz + 2 * L->R->nnz : 2 * sweeps * L->nnz;
			}
			return;
		}
		if( !L->coarser ) {
			symmetric_enqueue( L, z, r, sweeps, zero_guess, fuse_rz );
			if( count_stats ) {
				L->stats.nnz_visited += 2 * sweeps * L->nnz;
			}
			return;
		}
		if( !ctx->fused_transfers || !L->is_stencil ) {
			// the reference's composition, primitive by primitive (multigrid.hpp:94-111)
			symmetric_enqueue( L, z, r, sweeps );
			op_mxv( L->f.get(), nullptr, L->A.get(), z, SLAB_DESC_NONE ); // f <- A z
			op_waxpby( L->f.get(), 1.0, r, -1.0, L->f.get() );            // f <- r - f
			op_mxv( L->r_c.get(), nullptr, L->R.get(), L->f.get(), SLAB_DESC_NONE );
			op_set_all( L->z_c.get(), 0.0 );
			mg_vcycle_enqueue( L->coarser.get(), L->z_c.get(), L->r_c.get(), sweeps, count_stats );
			op_mxv( L->f.get(), nullptr, L->R.get(), L->z_c.get(), SLAB_DESC_TRANSPOSE );
			op_waxpby( z, 1.0, z, 1.0, L->f.get() );
			symmetric_enqueue( L, z, r, sweeps );
		} else {
			// Fused transfers. On a stencil level colour 0 is exactly the injected rows, in coarse-index
			// order. The residual + restriction (and the zeroing of the coarse guess) ride on the LAST
			// colour step of the pre-smoother — backward, colour 0, every other colour final — when that
			// launch keeps its matrix rows in registers, else they are one extra pass over the colour-0
			// rows; the prolongation rides on the FIRST colour step of the post-smoother (forward, colour
			// 0), which reads no other colour-0 value. Results are bit-identical to the composition above.
			const bool fuse_residual = planes_usable( L ) || kern::gs_color_step_can_fuse_residual( L->colorA, static_cast< int64_t >( L->color_size[ 0 ] ) );
			const bool ghosts = L->z_c->n_alloc > L->z_c->n; // distributed: the ghost tail must be zeroed too
			for( uint64_t sweep = 0; sweep < sweeps; ++sweep ) {
				sweep_pair_enqueue( L, z, r, sweep == 0 && zero_guess && planes_usable( L ) ? 8 : 0, sweep + 1 == sweeps && fuse_residual ? 2 : 0 );
			}
			if( ctx->after_presmooth ) { // cg.cu: side work that belongs under the coarse levels (taken once, by the finest level)
				std::function< void() > side;
				side.swap( ctx->after_presmooth );
				side();
			}
			if( !fuse_residual ) {
				kern::residual_restrict( ctx->stream, L->colorA, L->d_rows,
					static_cast< int64_t >( L->r_c->n ), z->d, r->d, L->r_c->d, L->z_c->d );
			}
			if( ghosts ) {
				op_set_all( L->z_c.get(), 0.0 );
			}
			mg_vcycle_enqueue( L->coarser.get(), L->z_c.get(), L->r_c.get(), sweeps, count_stats, true ); // z_c was zeroed above
			for( uint64_t sweep = 0; sweep < sweeps; ++sweep ) {
				sweep_pair_enqueue( L, z, r, sweep == 0 ? 1 : 0, sweep + 1 == sweeps && fuse_rz && planes_usable( L ) ? 16 : 0 );
			}
		}
		if( count_stats ) {
			L->stats.nnz_visited += 4 * sweeps * L->nnz + L->nnz + 2 * L->R->nnz;
		}
	}

	void mg_vcycle( slab_level_s * L, slab_vec_s * z, slab_vec_s * r, uint64_t sweeps ) {
		if( z->n != L->n || r->n != L->n ) { // multigrid.hpp:89-91
			fail( SLAB_ERR_DIMENSION_MISMATCH, "mg_vcycle: vector lengths differ from the level size" );
		}
		if( sweeps < 1 ) {
			fail( SLAB_ERR_INVALID_ARGUMENT, "SmootherConfig: sweeps must be at least 1" );
		}
		slab_ctx_s * ctx = L->ctx;
		ctx->after_presmooth = nullptr; // only cg.cu hands the V-cycle side work (a solve that threw may have left it behind)
		mg_vcycle_prepare( L, z, r, sweeps ); // allocations and uploads happen before any capture
		if( !ctx->use_graphs || ctx->profiling ) {
			halo_exchange( L, z, -1 ); // the caller's z: ghost copies may be stale
			mg_vcycle_enqueue( L, z, r, sweeps, true );
			return;
		}
		if( L->vcycle_exec == nullptr || L->vcycle_z != z->d || L->vcycle_r != r->d || L->vcycle_sweeps != sweeps
			|| L->vcycle_fused != ctx->fused_transfers || L->vcycle_epoch != g_tuning_epoch || L->vcycle_scratch != ctx->scratch_gen ) {
			if( L->vcycle_exec ) {
				cudaGraphExecDestroy( L->vcycle_exec );
				L->vcycle_exec = nullptr;
			}
			cudaGraph_t graph = nullptr;
			const uint64_t launches_before = thread_launches();
			SLAB_CUDA( cudaStreamBeginCapture( ctx->stream, halo_has_comm( ctx ) ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeThreadLocal ) );
			try {
				halo_exchange( L, z, -1 );
				mg_vcycle_enqueue( L, z, r, sweeps, false );
			} catch( ... ) {
				cudaStreamEndCapture( ctx->stream, &graph );
				if( graph ) {
					cudaGraphDestroy( graph );
				}
				throw;
			}
			SLAB_CUDA( cudaStreamEndCapture( ctx->stream, &graph ) );
			L->vcycle_launches = thread_launches() - launches_before;
			g_launch_count -= L->vcycle_launches; // enqueued into the graph, not launched
			thread_launches() = launches_before;
			const cudaError_t err = cudaGraphInstantiate( &L->vcycle_exec, graph, 0 );
			cudaGraphDestroy( graph );
			SLAB_CUDA( err );
			L->vcycle_z = z->d;
			L->vcycle_r = r->d;
			L->vcycle_sweeps = sweeps;
			L->vcycle_fused = ctx->fused_transfers;
			L->vcycle_epoch = g_tuning_epoch;
			L->vcycle_scratch = ctx->scratch_gen;
		}
		SLAB_CUDA( cudaGraphLaunch( L->vcycle_exec, ctx->stream ) );
		count_launch( L->vcycle_launches );
		vcycle_stats( L, sweeps );
	}

} // namespace slabgpu
