// tile.cu — fine-level kernels that stage the gathered vector through shared memory with bulk-async copies.
//
// Why. The dictionary-coded kernels of packed.cu issue one L1 request per stored entry (27 per row); on the
// fine levels they are bound by the L2 -> L1 path: every colour step pulls the whole vector through it (each
// warp fetches its own 3x3 neighbourhood of x-lines, 146 MB per 192^3 colour step against 57 MB of vector),
// and nothing but registers holds the bytes in flight. This file removes both limits for matrices whose rows
// live on a 3D box (the multigrid levels of the benchmark):
//
//  * the matrix stream shrinks once more: such a matrix is a subset-of-27-offsets matrix (BoxTile, common.hpp),
//    a row is a 32-bit mask over the 27 (offset, value) pairs — built from the coded rows entry by entry and
//    verified when the level is created, so nothing is assumed about where the matrix came from;
//  * a thread block owns TY row-lines (whole x-lines) and marches along z; the (2 TY + 1) x-lines of every
//    z-plane it needs are ONE contiguous range of the vector and arrive by one cp.async.bulk into a ring of
//    plane slabs in shared memory (mbarrier complete_tx), slabs ahead of the one being computed on. Every
//    vector element is fetched about once per launch and the gathers are conflict-free 16-byte shared-memory
//    reads;
//  * the two colours that differ only in the parity of x become ONE launch: colour 2p+1 reads colour 2p only
//    through the x-neighbours on its own line (every other neighbour line has another y- or z-parity), and
//    that line belongs to the same block, so a block-wide barrier between the two phases is the whole
//    dependency. The reference's colour order (smoother.hpp:80-82, 95-97) is kept row for row: each row sees
//    exactly the neighbour values it sees in the colour-by-colour sweep, and sums them in the same ascending
//    column order with separately rounded products (operations.hpp:116-125), so the results are bit-identical.
//    A thread owns the pair of rows (x, x+1) of a line: one aligned 16-byte read per neighbour line serves
//    both, and the new pair goes back to the vector as one 16-byte store.
#include "kernels.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "common.hpp"
#include "device_util.cuh"
#include "packed_decode.cuh"

namespace slabgpu {

	int g_use_tile = 1;
	int64_t g_tile_min_rows = 200000; // rows per colour pair / per product below which the per-row kernels stay
	int g_tile_ty = 0;
	int g_tile_cz = 0;
	int g_tile_ns = 0;

	void BoxTile::release() {
		if( masks ) {
			cudaFree( masks );
		}
		masks = nullptr;
		regular = false;
	}

	namespace kern {

		namespace {

			using namespace dev;

			constexpr unsigned int kAllBits = ( 1u << 27 ) - 1u;
			constexpr int kMaxThreads = 768;
			constexpr int kMaxSlots = 16;
			constexpr int kHeaderBytes = 128; // mbarriers in front of the slabs; also the landing zone of [x0 - 1] reads at x0 = 0

			// ------------------------------------------------------------ mbarrier / bulk-copy wrappers (PTX)

			__device__ __forceinline__ uint32_t smem_u32( const void * p ) {
				return static_cast< uint32_t >( __cvta_generic_to_shared( p ) );
			}
			__device__ __forceinline__ void mbar_init( uint64_t * bar, unsigned int count ) {
				asm volatile( "mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"( smem_u32( bar ) ), "r"( count ) : "memory" );
			}
			__device__ __forceinline__ void mbar_fence_init() {
				asm volatile( "fence.mbarrier_init.release.cluster;" ::: "memory" );
			}
			__device__ __forceinline__ void mbar_arrive_expect_tx( uint64_t * bar, unsigned int bytes ) {
				asm volatile( "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"( smem_u32( bar ) ), "r"( bytes ) : "memory" );
			}
			__device__ __forceinline__ void mbar_arrive( uint64_t * bar ) {
				asm volatile( "mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"( smem_u32( bar ) ) : "memory" );
			}
			__device__ __forceinline__ void mbar_wait( uint64_t * bar, unsigned int parity ) {
				asm volatile(
					"{\n"
					".reg .pred P1;\n"
					"LAB_WAIT:\n"
					"mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
					"@P1 bra DONE;\n"
					"bra LAB_WAIT;\n"
					"DONE:\n"
					"}" ::"r"( smem_u32( bar ) ),
					"r"( parity )
					: "memory" );
			}
			// global -> shared bulk copy (the TMA unit moves it; SASS: UBLKCP), completion counted on `bar`
			__device__ __forceinline__ void bulk_g2s( void * dst, const void * src, unsigned int bytes, uint64_t * bar ) {
				asm volatile( "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"( smem_u32( dst ) ),
					"l"( __cvta_generic_to_global( src ) ), "r"( bytes ), "r"( smem_u32( bar ) )
					: "memory" );
			}
			// generic-proxy accesses to shared memory before this point are ordered before later async-proxy ones
			__device__ __forceinline__ void fence_proxy_async() {
				asm volatile( "fence.proxy.async.shared::cta;" ::: "memory" );
			}

			// ------------------------------------------------------------ geometry of a launch

			struct BoxGeom {
				double v[ 27 ];    // value of each offset, slot = 9*(dz+1) + 3*(dy+1) + (dx+1)
				int lx, ly, lz;    // the box
				int hx;            // thread columns: lx / 2 (a thread owns x = 2 qx and 2 qx + 1)
				int sy, sz;        // row-lines / row-planes of the launch
				int py, pz;        // parity of their y and z (colour pairs); 0 for products
				int step;          // distance between row-lines: 2 (colour pairs) or 1 (products)
				int ty, cz, ns;    // row-lines per block, row-planes per block, ring slots
				int nyt;           // y tiles
				int nl;            // x-lines per slab: step*(ty-1) + 3
				long long pos0, pos1; // first position of the x-even / x-odd colour block (colour pairs)
			};

			// ------------------------------------------------------------ the ordered row sum from the slabs

			// c0, c1, c2: the thread's pair (x0, x0 + 1) on the row's own line in the planes z-1, z, z+1; the lines
			// y-1 and y+1 are lx doubles before and after. PAR: the row is x0 (0) or x0 + 1 (1). Ascending column
			// order = planes, then lines, then x (problem.hpp:108-127). FULL: all 27 entries stored (no tests).
			template< int PAR, bool FULL >
			__device__ __forceinline__ double box_row_sum( const double * c0, const double * c1, const double * c2, int lx, unsigned int m,
				const BoxGeom & G ) {
				double e[ 27 ];
				#pragma unroll
				for( int k = 0; k < 3; ++k ) {
					const double * c = k == 0 ? c0 : ( k == 1 ? c1 : c2 );
					#pragma unroll
					for( int dl = 0; dl < 3; ++dl ) {
						const double * q = c + ( dl - 1 ) * lx;
						const double2 pr = *reinterpret_cast< const double2 * >( q );
						const int s = 9 * k + 3 * dl;
						if( PAR == 0 ) {
							e[ s ] = q[ -1 ];
							e[ s + 1 ] = pr.x;
							e[ s + 2 ] = pr.y;
						} else {
							e[ s ] = pr.x;
							e[ s + 1 ] = pr.y;
							e[ s + 2 ] = q[ 2 ];
						}
					}
				}
				double acc = 0.0;
				#pragma unroll
				for( int s = 0; s < 27; ++s ) {
					const double prod = __dmul_rn( G.v[ s ], e[ s ] );
					if( FULL || ( ( m >> s ) & 1u ) ) { // a predicated add: absent entries add nothing
						acc = __dadd_rn( acc, prod );
					}
				}
				return acc;
			}

			// smoother.hpp:60-72 for one row of the pair: z_i <- ((r_i - s) + z_i d) / d, `passes` times in a row
			// (2: the turnaround of a symmetric sweep, smoother.hpp:108-111 — only z_i itself changes in between).
			// The new value goes into the slab: the other colour of the pair and the fused residual read it there.
			template< int PAR, bool FULL >
			__device__ __forceinline__ double gs_phase( const double * c0, double * c1, const double * c2, int lx, unsigned int m, double ri,
				double zi, const BoxGeom & G, int passes ) {
				const double d = G.v[ 13 ];
				#pragma unroll 1
				for( int pass = 0; pass < passes; ++pass ) {
					const double s = box_row_sum< PAR, FULL >( c0, c1, c2, lx, m, G );
					zi = __ddiv_rn( __dadd_rn( __dadd_rn( ri, -s ), __dmul_rn( zi, d ) ), d );
					c1[ PAR ] = zi;
				}
				return zi;
			}

			// ------------------------------------------------------------ the slab ring

			struct Ring {
				uint64_t * full;   // one mbarrier per slot
				double * slabs;    // slot s at slabs + s * slab_elems
				int slab_elems;
				int ns;
				__device__ __forceinline__ double * slot( int g ) const {
					return slabs + static_cast< size_t >( g % ns ) * slab_elems;
				}
				__device__ __forceinline__ void wait( int g ) const {
					mbar_wait( full + g % ns, static_cast< unsigned int >( ( g / ns ) & 1 ) );
				}
			};

			// slab g of a block = x-lines [ya, yb] of plane zp0 + g (one contiguous range of the vector); planes outside
			// the box are not loaded (their slab is only ever read for entries the masks rule out)
			__device__ __forceinline__ void ring_issue( const Ring & R, int g, const double * vec, const BoxGeom & G, int zp0, int yl0, int ya, int yb ) {
				uint64_t * bar = R.full + g % R.ns;
				const int zp = zp0 + g;
				if( zp < 0 || zp >= G.lz || yb < ya ) {
					mbar_arrive( bar );
					return;
				}
				const size_t elems = static_cast< size_t >( yb - ya + 1 ) * G.lx;
				const unsigned int bytes = static_cast< unsigned int >( elems * sizeof( double ) );
				mbar_arrive_expect_tx( bar, bytes );
				double * dst = R.slot( g ) + static_cast< size_t >( ya - yl0 ) * G.lx;
				const double * src = vec + ( static_cast< size_t >( zp ) * G.ly + ya ) * G.lx;
				constexpr unsigned int kPiece = 32768;
				for( unsigned int off = 0; off < bytes; off += kPiece ) {
					const unsigned int len = bytes - off < kPiece ? bytes - off : kPiece;
					bulk_g2s( reinterpret_cast< char * >( dst ) + off, reinterpret_cast< const char * >( src ) + off, len, bar );
				}
			}

			// ------------------------------------------------------------ colour pair: smoother.hpp:60-113

			// MODE 0: forward — the x-even colour, then the x-odd one (colours 2p, 2p+1 of smoother.hpp:80-82);
			// MODE 1: backward — x-odd, then x-even (smoother.hpp:95-97);
			// MODE 2: the turnaround of a symmetric sweep — even, odd, odd, even (colours 6,7,7,6).
			// flags bit 0 (MODE 0, colour 0 only): prolongation in front, z_i <- 1 z_i + 1 (0 + 1 src[p]) (multigrid.hpp:71-81);
			// flags bit 1 (MODE 1, colour 0 only): residual + restriction behind, out[p] = 0 + 1 (1 r_i + (-1)(A z)_i),
			// zero[p] = 0 (multigrid.hpp:100-104); p = position inside the colour-0 block = coarse row.
			template< int MODE >
			__global__ void __launch_bounds__( kMaxThreads, 1 ) k_gs_pair_tile( const uint32_t * __restrict__ masks,
				const __grid_constant__ BoxGeom G, double * z, const double * r, int flags, const double * src, double * out, double * zero ) {
				extern __shared__ __align__( 128 ) unsigned char smem_raw[];
				Ring R;
				R.full = reinterpret_cast< uint64_t * >( smem_raw );
				R.slabs = reinterpret_cast< double * >( smem_raw + kHeaderBytes );
				R.slab_elems = G.nl * G.lx;
				R.ns = G.ns;

				const int t = threadIdx.x;
				const int tyi = t / G.hx;
				const int qx = t - tyi * G.hx;
				const int ytile = blockIdx.x % G.nyt;
				const int chunk = blockIdx.x / G.nyt;
				const int jy = ytile * G.ty + tyi;
				const bool valid = tyi < G.ty && jy < G.sy;
				const int zc0 = chunk * G.cz;
				const int czc = min( G.cz, G.sz - zc0 );
				const int nslabs = 2 * czc + 1;
				const int yl0 = G.py + 2 * ytile * G.ty - 1;     // first x-line of a slab
				const int ya = max( yl0, 0 );
				const int yb = min( yl0 + G.nl - 1, G.ly - 1 );
				const int zp0 = G.pz + 2 * zc0 - 1;              // plane of slab 0
				const int lx = G.lx;

				if( t == 0 ) {
					for( int s = 0; s < G.ns; ++s ) {
						mbar_init( R.full + s, 1u );
					}
					mbar_fence_init();
				}
				// immutable data first: the masks of the first step (the previous kernel may still be running)
				const long long line_off = qx + static_cast< long long >( G.hx ) * jy; // + hx*sy*jz
				const long long plane_rows = static_cast< long long >( G.hx ) * G.sy;
				unsigned int m0 = kAllBits, m1 = kAllBits;
				if( valid ) {
					m0 = masks[ G.pos0 + line_off + plane_rows * zc0 ];
					m1 = masks[ G.pos1 + line_off + plane_rows * zc0 ];
				}
				__syncthreads();
				dep_trigger();
				dep_wait();
				if( t == 0 ) {
					const int first = min( G.ns, nslabs );
					for( int g = 0; g < first; ++g ) {
						ring_issue( R, g, z, G, zp0, yl0, ya, yb );
					}
				}
				const int y = G.py + 2 * jy;
				const size_t slab_line = static_cast< size_t >( 1 + 2 * tyi ) * lx + 2 * qx; // the pair on the row's own line
				double2 rr = make_double2( 0.0, 0.0 );
				size_t i0 = 0;
				if( valid ) {
					i0 = ( static_cast< size_t >( G.pz + 2 * zc0 ) * G.ly + y ) * lx + 2 * qx;
					rr = *reinterpret_cast< const double2 * >( r + i0 );
				}
				#pragma unroll 1
				for( int j = 0; j < czc; ++j ) {
					// the next step's masks and right-hand sides travel while this step computes
					unsigned int m0n = kAllBits, m1n = kAllBits;
					double2 rrn = make_double2( 0.0, 0.0 );
					const size_t i0n = i0 + 2 * static_cast< size_t >( G.ly ) * lx;
					if( valid && j + 1 < czc ) {
						m0n = masks[ G.pos0 + line_off + plane_rows * ( zc0 + j + 1 ) ];
						m1n = masks[ G.pos1 + line_off + plane_rows * ( zc0 + j + 1 ) ];
						rrn = *reinterpret_cast< const double2 * >( r + i0n );
					}
					R.wait( 2 * j );
					R.wait( 2 * j + 1 );
					R.wait( 2 * j + 2 );
					const double * c0 = R.slot( 2 * j ) + slab_line;
					double * c1 = R.slot( 2 * j + 1 ) + slab_line;
					const double * c2 = R.slot( 2 * j + 2 ) + slab_line;
					const bool full = __all_sync( 0xffffffffu, m0 == kAllBits && m1 == kAllBits );
					double z0 = 0.0, z1 = 0.0;
					const long long p = line_off + plane_rows * ( zc0 + j ); // position inside a colour block
					if( valid ) {
						const double2 zz = *reinterpret_cast< const double2 * >( c1 );
						z0 = zz.x;
						z1 = zz.y;
					}
					if( MODE == 0 || MODE == 2 ) {
						if( valid ) {
							if( MODE == 0 && ( flags & 1 ) ) {
								const double f = __dadd_rn( 0.0, __dmul_rn( 1.0, src[ p ] ) );
								z0 = __dadd_rn( __dmul_rn( 1.0, z0 ), __dmul_rn( 1.0, f ) );
								c1[ 0 ] = z0; // the row sum reads the row's own entry from the slab
							}
							z0 = full ? gs_phase< 0, true >( c0, c1, c2, lx, m0, rr.x, z0, G, 1 ) : gs_phase< 0, false >( c0, c1, c2, lx, m0, rr.x, z0, G, 1 );
						}
						__syncthreads();
						if( valid ) {
							const int passes = MODE == 2 ? 2 : 1;
							z1 = full ? gs_phase< 1, true >( c0, c1, c2, lx, m1, rr.y, z1, G, passes ) : gs_phase< 1, false >( c0, c1, c2, lx, m1, rr.y, z1, G, passes );
						}
						if( MODE == 2 ) {
							__syncthreads();
							if( valid ) {
								z0 = full ? gs_phase< 0, true >( c0, c1, c2, lx, m0, rr.x, z0, G, 1 ) : gs_phase< 0, false >( c0, c1, c2, lx, m0, rr.x, z0, G, 1 );
							}
						}
					} else {
						if( valid ) {
							z1 = full ? gs_phase< 1, true >( c0, c1, c2, lx, m1, rr.y, z1, G, 1 ) : gs_phase< 1, false >( c0, c1, c2, lx, m1, rr.y, z1, G, 1 );
						}
						__syncthreads();
						if( valid ) {
							z0 = full ? gs_phase< 0, true >( c0, c1, c2, lx, m0, rr.x, z0, G, 1 ) : gs_phase< 0, false >( c0, c1, c2, lx, m0, rr.x, z0, G, 1 );
							if( flags & 2 ) {
								const double az = full ? box_row_sum< 0, true >( c0, c1, c2, lx, m0, G ) : box_row_sum< 0, false >( c0, c1, c2, lx, m0, G );
								const double f = __dadd_rn( __dmul_rn( 1.0, rr.x ), __dmul_rn( -1.0, az ) );
								out[ p ] = __dadd_rn( 0.0, __dmul_rn( 1.0, f ) );
								zero[ p ] = 0.0;
							}
						}
					}
					if( valid ) {
						*reinterpret_cast< double2 * >( z + i0 ) = make_double2( z0, z1 );
					}
					// the two oldest slabs are done with: their slots take the slabs ns ahead
					fence_proxy_async();
					__syncthreads();
					if( t == 0 ) {
						if( 2 * j + G.ns < nslabs ) {
							ring_issue( R, 2 * j + G.ns, z, G, zp0, yl0, ya, yb );
						}
						if( 2 * j + 1 + G.ns < nslabs ) {
							ring_issue( R, 2 * j + 1 + G.ns, z, G, zp0, yl0, ya, yb );
						}
					}
					m0 = m0n;
					m1 = m1n;
					rr = rrn;
					i0 = i0n;
				}
			}

			// ------------------------------------------------------------ building and checking the masks

			// one thread per row position: the row's codes -> mask, every entry checked against the offset table;
			// anything that does not fit (escaped row, offset outside the 27, another value for an offset, an
			// offset that leaves the box, no diagonal, a row index that is not where the lattice puts it) counts as bad
			template< int CHUNKS >
			__global__ void __launch_bounds__( kBlock ) k_box_masks( const uint4 * __restrict__ codes, int ncodes, const DictEntry * __restrict__ dict,
				int dict_size, const int32_t * __restrict__ rows, int64_t npos, int lx, int ly, int lz, const double * __restrict__ canon,
				uint32_t * __restrict__ masks, unsigned long long * bad ) {
				const int64_t pos = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( pos >= npos ) {
					return;
				}
				const int64_t i = rows != nullptr ? static_cast< int64_t >( rows[ pos ] ) : pos;
				if( i < 0 ) {
					masks[ pos ] = 0u;
					return;
				}
				coded::RowCodes< CHUNKS > rc;
				coded::codes_load( codes, pos, rc );
				bool ok = !rc.escaped();
				const int x = static_cast< int >( i % lx ), y = static_cast< int >( ( i / lx ) % ly ), zc = static_cast< int >( i / ( static_cast< int64_t >( lx ) * ly ) );
				ok = ok && zc < lz;
				unsigned int m = 0u;
				const int64_t plane = static_cast< int64_t >( lx ) * ly;
				for( int k = 0; k < ncodes && ok; ++k ) {
					const unsigned int code = ( rc.word( k >> 2 ) >> ( 8 * ( k & 3 ) ) ) & 0xffu;
					if( code == 0u ) {
						continue;
					}
					if( static_cast< int >( code ) >= dict_size ) {
						ok = false;
						break;
					}
					const int64_t tt = static_cast< int64_t >( dict[ code ].delta ) + 1 + lx + plane;
					if( tt < 0 ) {
						ok = false;
						break;
					}
					const int64_t dz = tt / plane, rem = tt % plane;
					const int64_t dy = rem / lx, dx = rem % lx;
					if( dz > 2 || dy > 2 || dx > 2 ) {
						ok = false;
						break;
					}
					const int s = static_cast< int >( 9 * dz + 3 * dy + dx );
					const int nx = x + static_cast< int >( dx ) - 1, ny = y + static_cast< int >( dy ) - 1, nz = zc + static_cast< int >( dz ) - 1;
					if( nx < 0 || nx >= lx || ny < 0 || ny >= ly || nz < 0 || nz >= lz ) {
						ok = false;
						break;
					}
					if( __double_as_longlong( dict[ code ].val ) != __double_as_longlong( canon[ s ] ) || ( ( m >> s ) & 1u ) || ( m >> s ) != 0u ) {
						ok = false; // another value for this offset, a repeated offset, or columns out of order
						break;
					}
					m |= 1u << s;
				}
				ok = ok && ( ( m >> 13 ) & 1u );
				if( !ok ) {
					atomicAdd( bad, 1ull );
					m = 0u;
				}
				masks[ pos ] = m;
			}

			// does every row store exactly the offsets that stay inside the box? (plane.cu runs without masks then)
			__global__ void __launch_bounds__( kBlock ) k_box_regular( const uint32_t * __restrict__ masks, const int32_t * __restrict__ rows, int64_t npos,
				int lx, int ly, int lz, unsigned long long * bad ) {
				const int64_t pos = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( pos >= npos ) {
					return;
				}
				const int64_t i = rows != nullptr ? static_cast< int64_t >( rows[ pos ] ) : pos;
				if( i < 0 ) {
					return;
				}
				const int x = static_cast< int >( i % lx ), y = static_cast< int >( ( i / lx ) % ly ), zc = static_cast< int >( i / ( static_cast< int64_t >( lx ) * ly ) );
				unsigned int m = 0u;
				for( int dz = -1; dz <= 1; ++dz ) {
					for( int dy = -1; dy <= 1; ++dy ) {
						for( int dx = -1; dx <= 1; ++dx ) {
							const int nx = x + dx, ny = y + dy, nz = zc + dz;
							if( nx >= 0 && nx < lx && ny >= 0 && ny < ly && nz >= 0 && nz < lz ) {
								m |= 1u << ( 9 * ( dz + 1 ) + 3 * ( dy + 1 ) + ( dx + 1 ) );
							}
						}
					}
				}
				if( masks[ pos ] != m ) {
					atomicAdd( bad, 1ull );
				}
			}

			// is the colour-major row list the parity lattice the pair kernel computes positions from?
			// position color_pos[c] + qx + sx (qy + sy qz)  <->  row (px + 2 qx) + lx ((py + 2 qy) + ly (pz + 2 qz))
			struct LatticeParam {
				long long color_pos[ 9 ];
				int lx, ly, lz;
			};
			__global__ void __launch_bounds__( kBlock ) k_box_lattice_check( const int32_t * __restrict__ rows, const LatticeParam L, unsigned long long * bad ) {
				const int64_t pos = static_cast< int64_t >( blockIdx.x ) * blockDim.x + threadIdx.x;
				if( pos >= L.color_pos[ 8 ] ) {
					return;
				}
				int c = 0;
				while( c < 7 && pos >= L.color_pos[ c + 1 ] ) {
					++c;
				}
				const int px = c & 1, py = ( c >> 1 ) & 1, pz = ( c >> 2 ) & 1;
				const int sx = count_parity( 0, L.lx, px ), sy = count_parity( 0, L.ly, py ), sz = count_parity( 0, L.lz, pz );
				const int64_t q = pos - L.color_pos[ c ];
				int32_t expect = -1;
				if( q < static_cast< int64_t >( sx ) * sy * sz ) {
					const int qx = static_cast< int >( q % sx ), qy = static_cast< int >( ( q / sx ) % sy ), qz = static_cast< int >( q / ( static_cast< int64_t >( sx ) * sy ) );
					expect = static_cast< int32_t >( ( px + 2 * qx ) + static_cast< int64_t >( L.lx ) * ( ( py + 2 * qy ) + static_cast< int64_t >( L.ly ) * ( pz + 2 * qz ) ) );
				}
				if( rows[ pos ] != expect ) {
					atomicAdd( bad, 1ull );
				}
			}

			template< class... KArgs, class... Args >
			void launch_pdl_smem( void ( *kernel )( KArgs... ), unsigned int grid, unsigned int block, size_t smem, cudaStream_t st, Args... args ) {
				cudaLaunchConfig_t cfg{};
				cfg.gridDim = dim3( grid, 1, 1 );
				cfg.blockDim = dim3( block, 1, 1 );
				cfg.dynamicSmemBytes = smem;
				cfg.stream = st;
				cudaLaunchAttribute attr[ 1 ];
				unsigned int count = 0;
				if( g_use_pdl ) {
					attr[ count ].id = cudaLaunchAttributeProgrammaticStreamSerialization;
					attr[ count ].val.programmaticStreamSerializationAllowed = 1;
					++count;
				}
				cfg.attrs = attr;
				cfg.numAttrs = count;
				SLAB_CUDA( cudaLaunchKernelEx( &cfg, kernel, static_cast< KArgs >( args )... ) );
				count_launch();
			}

			constexpr size_t kSmemLimit = 227u * 1024u;

			template< int MODE >
			void allow_big_smem() {
				static bool done = false; // per kernel symbol; the attribute is per device function, set once
				if( !done ) {
					SLAB_CUDA( cudaFuncSetAttribute( k_gs_pair_tile< MODE >, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast< int >( kSmemLimit ) ) );
					done = true;
				}
			}

			// tile shape of a launch over sy row-lines and sz row-planes (lines `step` apart); false: nothing fits
			bool choose_shape( BoxGeom & G, int sm_count ) {
				const int line_bytes = G.lx * 8;
				int best_ty = 0;
				for( int ty : { 8, 4, 2, 1 } ) {
					if( g_tile_ty > 0 && ty != g_tile_ty ) {
						continue;
					}
					if( G.hx * ty > ( g_tile_ty > 0 ? kMaxThreads : 512 ) ) {
						continue;
					}
					const int nl = G.step * ( ty - 1 ) + 3;
					// at least 5 slots, two blocks per SM
					if( static_cast< size_t >( 5 ) * nl * line_bytes + kHeaderBytes + 16 > kSmemLimit / 2 && g_tile_ty == 0 ) {
						continue;
					}
					// enough blocks to fill the GPU twice, if the launch is large enough for that at all
					const int nyt = ( G.sy + ty - 1 ) / ty;
					if( g_tile_ty == 0 && ty > 1 && static_cast< int64_t >( nyt ) * ( ( G.sz + 3 ) / 4 ) < 2 * sm_count ) {
						continue;
					}
					best_ty = ty;
					break;
				}
				if( best_ty == 0 ) {
					return false;
				}
				G.ty = best_ty;
				G.nl = G.step * ( best_ty - 1 ) + 3;
				G.nyt = ( G.sy + best_ty - 1 ) / best_ty;
				// row-planes per block: as long a march as still leaves two blocks per SM
				int cz = g_tile_cz > 0 ? g_tile_cz : 16;
				while( g_tile_cz == 0 && cz > 2 && static_cast< int64_t >( G.nyt ) * ( ( G.sz + cz - 1 ) / cz ) < 2 * sm_count ) {
					cz /= 2;
				}
				G.cz = std::min( cz, G.sz );
				const size_t slab_bytes = static_cast< size_t >( G.nl ) * line_bytes;
				int ns = g_tile_ns > 0 ? g_tile_ns : 7;
				const size_t budget = kSmemLimit / 2 - kHeaderBytes - 16;
				while( ns > 5 && ns * slab_bytes > budget ) {
					--ns;
				}
				ns = std::min( ns, kMaxSlots );
				if( ns < 4 || ns * slab_bytes + kHeaderBytes + 16 > kSmemLimit ) {
					return false;
				}
				G.ns = ns;
				return true;
			}

			size_t smem_bytes( const BoxGeom & G ) {
				return static_cast< size_t >( kHeaderBytes ) + static_cast< size_t >( G.ns ) * G.nl * G.lx * 8 + 16;
			}

		} // namespace

		bool gs_pair_tile_usable( const BoxTile & T, int64_t pair_rows ) {
			return g_use_tile && T.usable() && pair_rows >= g_tile_min_rows && ( T.lx % 2 ) == 0 && T.lx >= 4 && T.ly >= 4 && T.lz >= 4;
		}

		// one launch for the colours (2 pair, 2 pair + 1): mode 0 forward, 1 backward, 2 turnaround
		void gs_pair_tile( cudaStream_t st, int sm_count, const BoxTile & T, const std::vector< int64_t > & color_pos, int pair, int mode, double * z,
			const double * r, int flags, const double * src, double * out, double * zero ) {
			BoxGeom G{};
			std::memcpy( G.v, T.vals, sizeof( G.v ) );
			G.lx = T.lx;
			G.ly = T.ly;
			G.lz = T.lz;
			G.hx = T.lx / 2;
			G.py = pair & 1;
			G.pz = ( pair >> 1 ) & 1;
			G.sy = count_parity( 0, T.ly, G.py );
			G.sz = count_parity( 0, T.lz, G.pz );
			G.step = 2;
			G.pos0 = color_pos[ 2 * pair ];
			G.pos1 = color_pos[ 2 * pair + 1 ];
			if( G.sy == 0 || G.sz == 0 ) {
				return;
			}
			if( !choose_shape( G, sm_count ) ) {
				fail( SLAB_ERR_INTERNAL, "gs_pair_tile: no tile shape fits this level" );
			}
			const unsigned int block = static_cast< unsigned int >( ( G.hx * G.ty + 31 ) / 32 * 32 );
			const unsigned int grid = static_cast< unsigned int >( G.nyt ) * static_cast< unsigned int >( ( G.sz + G.cz - 1 ) / G.cz );
			const size_t smem = smem_bytes( G );
			switch( mode ) {
				case 0:
					allow_big_smem< 0 >();
					launch_pdl_smem( k_gs_pair_tile< 0 >, grid, block, smem, st, T.masks, G, z, r, flags, src, out, zero );
					break;
				case 1:
					allow_big_smem< 1 >();
					launch_pdl_smem( k_gs_pair_tile< 1 >, grid, block, smem, st, T.masks, G, z, r, flags, src, out, zero );
					break;
				default:
					allow_big_smem< 2 >();
					launch_pdl_smem( k_gs_pair_tile< 2 >, grid, block, smem, st, T.masks, G, z, r, flags, src, out, zero );
			}
		}

	} // namespace kern

	// ---------------------------------------------------------------- building the masks

	bool box_tile_lattice_ok( slab_ctx_s * ctx, const int32_t * d_rows, const std::vector< int64_t > & color_pos, const Decomp & D ) {
		using namespace kern;
		if( color_pos.size() != 9 || d_rows == nullptr ) {
			return false;
		}
		LatticeParam L{};
		for( int c = 0; c < 9; ++c ) {
			L.color_pos[ c ] = color_pos[ c ];
		}
		L.lx = D.l[ 0 ];
		L.ly = D.l[ 1 ];
		L.lz = D.l[ 2 ];
		unsigned long long * d_bad = nullptr;
		unsigned long long bad = 1;
		SLAB_CUDA( cudaMalloc( &d_bad, sizeof( unsigned long long ) ) );
		cudaStream_t st = ctx->stream;
		cudaError_t err = cudaMemsetAsync( d_bad, 0, sizeof( unsigned long long ), st );
		if( err == cudaSuccess && color_pos[ 8 ] > 0 ) {
			k_box_lattice_check<<< dev::blocks_for( color_pos[ 8 ] ), dev::kBlock, 0, st >>>( d_rows, L, d_bad );
			count_launch();
			err = cudaGetLastError();
		}
		if( err == cudaSuccess ) {
			err = cudaMemcpyAsync( &bad, d_bad, sizeof( bad ), cudaMemcpyDeviceToHost, st );
		}
		if( err == cudaSuccess ) {
			err = cudaStreamSynchronize( st );
		}
		cudaFree( d_bad );
		SLAB_CUDA( err );
		return bad == 0;
	}

	void box_tile_build( slab_ctx_s * ctx, const Sell & S, const int32_t * d_rows, const Decomp & D, BoxTile & T ) {
		using namespace kern;
		T.release();
		const Packed & P = S.packed;
		if( !g_use_tile || !P.usable() || P.escaped_rows != 0 || D.n_ghost != 0 || P.chunks > 2 ) {
			return;
		}
		const int lx = D.l[ 0 ], ly = D.l[ 1 ], lz = D.l[ 2 ];
		if( lx < 4 || ly < 4 || lz < 4 ) {
			return; // offsets would be ambiguous on thinner boxes
		}
		// the offset table from the dictionary: one value per offset, every offset one of the 27
		double canon[ 27 ] = { 0.0 };
		bool seen[ 27 ] = { false };
		const int64_t plane = static_cast< int64_t >( lx ) * ly;
		for( int t = 1; t < P.dict_size; ++t ) {
			const int64_t tt = static_cast< int64_t >( P.h_dict[ t ].delta ) + 1 + lx + plane;
			if( tt < 0 ) {
				return;
			}
			const int64_t dz = tt / plane, rem = tt % plane, dy = rem / lx, dx = rem % lx;
			if( dz > 2 || dy > 2 || dx > 2 ) {
				return;
			}
			const int s = static_cast< int >( 9 * dz + 3 * dy + dx );
			if( seen[ s ] ) {
				return; // two values on one offset: not this kind of matrix
			}
			seen[ s ] = true;
			canon[ s ] = P.h_dict[ t ].val;
		}
		if( !seen[ 13 ] || canon[ 13 ] == 0.0 ) {
			return;
		}
		const int64_t npos = S.nslices * kSlice;
		double * d_canon = nullptr;
		unsigned long long * d_bad = nullptr;
		unsigned long long bad = 1;
		cudaStream_t st = ctx->stream;
		try {
			SLAB_CUDA( cudaMalloc( &T.masks, std::max< int64_t >( npos, 1 ) * sizeof( uint32_t ) ) );
			SLAB_CUDA( cudaMalloc( &d_canon, sizeof( canon ) ) );
			SLAB_CUDA( cudaMalloc( &d_bad, sizeof( unsigned long long ) ) );
			upload_sync( st, d_canon, canon, sizeof( canon ) );
			SLAB_CUDA( cudaMemsetAsync( d_bad, 0, sizeof( unsigned long long ), st ) );
			SLAB_CUDA( cudaMemsetAsync( T.masks, 0, std::max< int64_t >( npos, 1 ) * sizeof( uint32_t ), st ) );
			const int64_t live = std::min< int64_t >( npos, S.nrows );
			if( P.chunks == 1 ) {
				k_box_masks< 1 ><<< dev::blocks_for( live ), dev::kBlock, 0, st >>>( P.codes, P.ncodes, P.dict, P.dict_size, d_rows, live, lx, ly, lz, d_canon, T.masks, d_bad );
			} else {
				k_box_masks< 2 ><<< dev::blocks_for( live ), dev::kBlock, 0, st >>>( P.codes, P.ncodes, P.dict, P.dict_size, d_rows, live, lx, ly, lz, d_canon, T.masks, d_bad );
			}
			SLAB_CUDA( cudaGetLastError() );
			count_launch();
			SLAB_CUDA( cudaMemcpyAsync( &bad, d_bad, sizeof( bad ), cudaMemcpyDeviceToHost, st ) );
			SLAB_CUDA( cudaStreamSynchronize( st ) );
		} catch( ... ) {
			cudaFree( d_canon );
			cudaFree( d_bad );
			T.release();
			throw;
		}
		cudaFree( d_canon );
		if( bad != 0 ) {
			cudaFree( d_bad );
			T.release();
			return;
		}
		// regular: every row stores exactly its in-box offsets, every value is finite (0 * value must be a zero)
		bool finite = true;
		for( int s = 0; s < 27; ++s ) {
			finite = finite && seen[ s ] && std::isfinite( canon[ s ] );
		}
		T.regular = false;
		if( finite ) {
			unsigned long long irregular = 1;
			cudaError_t err = cudaMemsetAsync( d_bad, 0, sizeof( unsigned long long ), st );
			if( err == cudaSuccess ) {
				k_box_regular<<< dev::blocks_for( std::min< int64_t >( npos, S.nrows ) ), dev::kBlock, 0, st >>>( T.masks, d_rows, std::min< int64_t >( npos, S.nrows ), lx, ly, lz, d_bad );
				count_launch();
				err = cudaGetLastError();
			}
			if( err == cudaSuccess ) {
				err = cudaMemcpyAsync( &irregular, d_bad, sizeof( irregular ), cudaMemcpyDeviceToHost, st );
			}
			if( err == cudaSuccess ) {
				err = cudaStreamSynchronize( st );
			}
			if( err != cudaSuccess ) {
				cudaFree( d_bad );
				T.release();
				SLAB_CUDA( err );
			}
			T.regular = irregular == 0;
		}
		cudaFree( d_bad );
		// (outside any stream capture: the launches themselves may be captured into graphs later)
		allow_big_smem< 0 >();
		allow_big_smem< 1 >();
		allow_big_smem< 2 >();
		std::memcpy( T.vals, canon, sizeof( canon ) );
		T.lx = lx;
		T.ly = ly;
		T.lz = lz;
	}

} // namespace slabgpu
